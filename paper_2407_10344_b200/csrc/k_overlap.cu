// k_overlap.cu -- voxel overlap counts (K2).
//
// "we define an overlap rate between two point clouds P_i and P_j as the
// fraction of points in P_i that fall within a voxel of P_j"; global
// factors for submap pairs whose overlap "exceeds a small threshold (e.g. 5%)".
//
// B200 design: one CTA per tile of consecutive source points
// of one pair; each thread streams only the 16 B {mu, C.xx} plane of the cloud,
// transforms in fp64 with the pinned fma order (bit-exact keys, Q10), probes
// one 16 B hash slot; hits are counted with __ballot_sync/__popc per warp and
// one integer atomicAdd per CTA (integer: exact and order-independent).
#include <cstdint>

#include "k_common.cuh"

namespace gvox {

namespace {

constexpr int kThreads = 256;
#ifndef GVOX_OVL_MINB
#define GVOX_OVL_MINB 7
#endif
// screening: sub-steps (256 points each) per decision window (one barrier each);
// (a power of two: windows <= 32 are slices of one 32-bit live-chunk word,
// larger ones several words)
#ifndef GVOX_OVL_WIN
#define GVOX_OVL_WIN 32
#endif
// screening: live chunks probed together per thread (2 or 4)
#ifndef GVOX_OVL_ILP
#define GVOX_OVL_ILP 4
#endif
#ifndef GVOX_OVL_LV_SMEM
#define GVOX_OVL_LV_SMEM 0
#endif
// exact chunk culling against the occupancy of the overlap's OWN level (1)
// instead of the coarsest level (0): also exact (a chunk whose transformed box
// meets no occupied cell of that level has no point in an occupied voxel of
// it), but measured slower at C5 (r02aj: screening 13.60 vs 12.54 ms -- at 1 m
// more chunk ranges exceed 3 cells per axis and go unculled, and the finer
// grid's cells are colder in L2), so the coarsest level stays
#ifndef GVOX_OVL_CULL_AT_LEVEL
#define GVOX_OVL_CULL_AT_LEVEL 0
#endif
#ifndef GVOX_OVL_CULL
#define GVOX_OVL_CULL 1
#endif
// screening without block barriers: warps publish (hits, points processed) into
// one packed 64-bit shared counter and stop on a certain decision (1), or the
// windowed block reductions (0)
#ifndef GVOX_OVL_NOBAR
#define GVOX_OVL_NOBAR 1
#endif

template <bool ALL_DENSE>
__global__ void __launch_bounds__(kThreads, GVOX_OVL_MINB)
    k_overlap(const CloudDev* const* __restrict__ clouds, const MapDev* const* __restrict__ maps,
              const PairDev* __restrict__ pairs, const int32_t* __restrict__ tile_start,
              const int32_t* __restrict__ tile_pair, int tile_pts, const double* __restrict__ poses,
              int level, int32_t* __restrict__ counts) {
  __shared__ double pose_s[24];
  __shared__ double R[9], t[3];
  __shared__ const float4* A_s;
  __shared__ int64_t range_s[2];
  __shared__ MapLevelDev lv_s;
  __shared__ int dyadic_s;
  __shared__ int warp_cnt[kThreads / 32];
  __shared__ float Rf[9], map_lo[4], map_hi[4];
  __shared__ const float* cbox_s;
  __shared__ MapLevelDev cv_s;  // culling level (GVOX_OVL_CULL_AT_LEVEL), used if dense
  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;
  const int32_t p = __ldg(tile_pair + tile);
  const PairDev pd = pairs[p];
  if (tid < 24) {
    pose_s[tid] = __ldg(poses + 12 * (int64_t)(tid < 12 ? pd.pi : pd.pj) + (tid % 12));
  } else if (tid == 32) {
    const CloudDev* cd = clouds[pd.src];
    int64_t b = (int64_t)(tile - __ldg(tile_start + p)) * tile_pts;
    int64_t e = b + tile_pts;
    A_s = cd->A;
    cbox_s = cd->chunk_box;
    range_s[0] = b;
    range_s[1] = e < cd->n ? e : cd->n;
  } else if (tid == 64) {
    const MapDev* md = maps[pd.tgt];
    lv_s = md->lv[level];
    dyadic_s = md->dyadic;
    for (int j = 0; j < 4; ++j) {
      map_lo[j] = md->box_lo[j];
      map_hi[j] = md->box_hi[j];
    }
    cv_s = md->lv[GVOX_OVL_CULL_AT_LEVEL ? level : md->levels - 1];
  }
  __syncthreads();
  if (tid == 0) {
    double v[3];
    relative_pose_dev(pose_s, pose_s + 12, R, t, v);
    for (int j = 0; j < 9; ++j) Rf[j] = (float)R[j];
  }
  __syncthreads();
  const MapLevelDev lv = lv_s;
  const int dyadic = dyadic_s;
  const float4* __restrict__ A = A_s;
  int cnt = 0;
  const int64_t kb = range_s[0], ke = range_s[1];
  const int warp = tid >> 5, lane = tid & 31;
  // Warp w owns tile chunks 8 m + w (32 consecutive points each), m < tile_pts /
  // 256 <= 32.  Exact chunk culling (k_common.cuh): one ballot marks the chunks
  // that cannot hit; the warp visits only the live ones, two at a time.
  const uint32_t cull =
      (GVOX_OVL_CULL && cbox_s)
          ? cull_ballot(cbox_s, (kb >> 5) + warp, kThreads / 32, (ke + 31) >> 5, Rf, t, map_lo,
                        map_hi, (cv_s.dense && cv_s.grid) ? &cv_s : nullptr)
          : 0u;
  const int nm = (int)((ke - kb + kThreads - 1) / kThreads);
  uint32_t live = ~cull & (nm >= 32 ? 0xffffffffu : ((1u << nm) - 1u));
  auto probe = [&](int m) -> int {
    const int64_t k = kb + (int64_t)m * kThreads + 32 * warp + lane;
    if (k >= ke) return 0;
    const float4 a = __ldg(A + pt_off(k));
    const double mx = a.x, my = a.y, mz = a.z;
    const double qx = __fma_rn(R[0], mx, __fma_rn(R[1], my, __fma_rn(R[2], mz, t[0])));
    const double qy = __fma_rn(R[3], mx, __fma_rn(R[4], my, __fma_rn(R[5], mz, t[1])));
    const double qz = __fma_rn(R[6], mx, __fma_rn(R[7], my, __fma_rn(R[8], mz, t[2])));
    const int32_t kx = voxel_coord0(qx, lv.r, lv.inv_r, dyadic);
    const int32_t ky = voxel_coord0(qy, lv.r, lv.inv_r, dyadic);
    const int32_t kz = voxel_coord0(qz, lv.r, lv.inv_r, dyadic);
    return lookup_level<ALL_DENSE>(lv, kx, ky, kz) >= 0;
  };
  while (live) {
    const int m0 = __ffs(live) - 1;
    live &= live - 1;
    if (live) {
      const int m1 = __ffs(live) - 1;
      live &= live - 1;
      cnt += probe(m0) + probe(m1);
    } else {
      cnt += probe(m0);
    }
  }
  // warp counts, then one atomic per CTA
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((tid & 31) == 0) warp_cnt[tid >> 5] = cnt;
  __syncthreads();
  if (tid == 0) {
    int s = 0;
    for (int w = 0; w < kThreads / 32; ++w) s += warp_cnt[w];
    if (s) atomicAdd(counts + p, s);
  }
}

// Screening decision (a factor for each pair whose overlap rate
// "exceeds a small threshold"): selected[p] = (count * den > n * num).  One CTA
// per pair walks its source points in blocks of kThreads * U and stops as soon
// as the decision is certain -- enough hits (count >= need) or too few points
// left to reach `need` -- so the decision equals the one from the exact count
// while accepted pairs cost only the points it takes to accept them.
template <bool ALL_DENSE>
__global__ void __launch_bounds__(kThreads, GVOX_OVL_MINB)
    k_overlap_select(const CloudDev* const* __restrict__ clouds,
                     const MapDev* const* __restrict__ maps, const PairDev* __restrict__ pairs,
                     const double* __restrict__ poses, int level, int32_t num, int32_t den,
                     uint8_t* __restrict__ selected) {
  __shared__ double pose_s[24];
  __shared__ double R[9], t[3];
  __shared__ const float4* A_s;
  __shared__ int64_t n_s;
  __shared__ MapLevelDev lv_s;
  __shared__ int dyadic_s;
  __shared__ int warp_cnt[2][kThreads / 32];
  __shared__ float Rf[9], map_lo[4], map_hi[4];
  __shared__ const float* cbox_s;
  __shared__ MapLevelDev cv_s;  // culling level (GVOX_OVL_CULL_AT_LEVEL), used if dense
  const int tid = threadIdx.x;
  const int32_t p = blockIdx.x;
  const PairDev pd = pairs[p];
  if (tid < 24) {
    pose_s[tid] = __ldg(poses + 12 * (int64_t)(tid < 12 ? pd.pi : pd.pj) + (tid % 12));
  } else if (tid == 32) {
    const CloudDev* cd = clouds[pd.src];
    A_s = cd->A;
    cbox_s = cd->chunk_box;
    n_s = cd->n;
  } else if (tid == 64) {
    const MapDev* md = maps[pd.tgt];
    lv_s = md->lv[level];
    dyadic_s = md->dyadic;
    for (int j = 0; j < 4; ++j) {
      map_lo[j] = md->box_lo[j];
      map_hi[j] = md->box_hi[j];
    }
    cv_s = md->lv[GVOX_OVL_CULL_AT_LEVEL ? level : md->levels - 1];
  }
  __syncthreads();
  if (tid == 0) {
    double v[3];
    relative_pose_dev(pose_s, pose_s + 12, R, t, v);
    for (int j = 0; j < 9; ++j) Rf[j] = (float)R[j];
  }
  __syncthreads();
#if GVOX_OVL_LV_SMEM
  const MapLevelDev& lv = lv_s;  // level descriptor read from shared memory (registers)
#else
  const MapLevelDev lv = lv_s;
#endif
  const int dyadic = dyadic_s;
  const float4* __restrict__ A = A_s;
  const int64_t n = n_s;
  const float* cbox = cbox_s;
  const int64_t nchunks = (n + 31) >> 5;
  // count * den > n * num  <=>  count >= need
  const int64_t need = (n * (int64_t)num) / den + 1;
  const int warp = tid >> 5, lane = tid & 31;
  auto probe = [&](int64_t m) -> int {
    const int64_t k = m * kThreads + 32 * warp + lane;
    if (k >= n) return 0;
    const float4 a = __ldg(A + pt_off(k));
    const double mx = a.x, my = a.y, mz = a.z;
    const double qx = __fma_rn(R[0], mx, __fma_rn(R[1], my, __fma_rn(R[2], mz, t[0])));
    const double qy = __fma_rn(R[3], mx, __fma_rn(R[4], my, __fma_rn(R[5], mz, t[1])));
    const double qz = __fma_rn(R[6], mx, __fma_rn(R[7], my, __fma_rn(R[8], mz, t[2])));
    const int32_t kx = voxel_coord0(qx, lv.r, lv.inv_r, dyadic);
    const int32_t ky = voxel_coord0(qy, lv.r, lv.inv_r, dyadic);
    const int32_t kz = voxel_coord0(qz, lv.r, lv.inv_r, dyadic);
    return lookup_level<ALL_DENSE>(lv, kx, ky, kz) >= 0;
  };
  // Windows of kWin sub-steps m (kThreads points each; warp w owns chunk 8 m + w):
  // each warp probes its live (non-culled) chunks of the window without
  // barriers, then one block reduction decides.  Culled chunks hold no hit.
  constexpr int kWin = GVOX_OVL_WIN;
  const int64_t msteps = (n + kThreads - 1) / kThreads;
  int64_t total = 0;
  int buf = 0;
  bool sel = false;
  uint32_t live = 0;  // bits for sub-steps mb .. mb + 31
  constexpr int kSub = kWin < 32 ? kWin : 32;  // sub-steps per live-word slice
  for (int64_t mw = 0; mw < msteps; mw += kWin) {
    int cnt = 0;
#pragma unroll 1
    for (int64_t mb = mw; mb < mw + kWin && mb < msteps; mb += kSub) {
      if ((mb & 31) == 0) {
        uint32_t cull = 0;
        if (GVOX_OVL_CULL && cbox)
          cull = cull_ballot(cbox, mb * (kThreads / 32) + warp, kThreads / 32, nchunks, Rf, t,
                             map_lo, map_hi, (cv_s.dense && cv_s.grid) ? &cv_s : nullptr);
        live = ~cull;
      }
      uint32_t w = (live >> (mb & 31)) & (kSub >= 32 ? 0xffffffffu : ((1u << (kSub & 31)) - 1u));
#if GVOX_OVL_ILP >= 4
      // up to four live chunks' lookups in flight per thread
      while (__popc(w) >= 4) {
        const int j0 = __ffs(w) - 1;
        w &= w - 1;
        const int j1 = __ffs(w) - 1;
        w &= w - 1;
        const int j2 = __ffs(w) - 1;
        w &= w - 1;
        const int j3 = __ffs(w) - 1;
        w &= w - 1;
        cnt += (probe(mb + j0) + probe(mb + j1)) + (probe(mb + j2) + probe(mb + j3));
      }
#endif
      while (w) {
        const int j0 = __ffs(w) - 1;
        w &= w - 1;
        if (w) {
          const int j1 = __ffs(w) - 1;
          w &= w - 1;
          cnt += probe(mb + j0) + probe(mb + j1);
        } else {
          cnt += probe(mb + j0);
        }
      }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) warp_cnt[buf][warp] = cnt;
    __syncthreads();
    int blk = 0;
#pragma unroll
    for (int q = 0; q < kThreads / 32; ++q) blk += warp_cnt[buf][q];
    buf ^= 1;  // double buffer: no second barrier needed before the next write
    total += blk;
    const int64_t done = (mw + kWin) * kThreads;
    const int64_t left = n - done;
    if (total >= need) {
      sel = true;
      break;
    }
    if (total + (left > 0 ? left : 0) < need) break;
  }
  if (tid == 0) selected[p] = sel ? 1 : 0;
}

// Barrier-free screening decision (same contract as k_overlap_select).  The
// CTA keeps ONE packed shared counter prog = hits << 32 | points processed;
// each warp walks its chunks (warp w owns chunk 8 m + w of sub-step m, the
// chunks of a 32-sub-step word culled together as above), probes up to four
// live chunks at a time, then adds its group's (hits, points) with a single
// shared atomicAdd -- culled chunks count as processed with no hit -- and
// reads back a consistent snapshot of both:
//   hits >= need                      -> selected (hits only grow),
//   hits + (n - processed) < need     -> rejected (every unprocessed point,
//                                        in flight in other warps or not yet
//                                        reached, could at most hit),
// so every decision is the one the exact count gives, and no warp waits at a
// barrier for the others.  A decided CTA's warps stop at their next check.
template <bool ALL_DENSE, bool DYADIC>
__global__ void __launch_bounds__(kThreads, GVOX_OVL_MINB)
    k_overlap_select_nb(const CloudDev* const* __restrict__ clouds,
                        const MapDev* const* __restrict__ maps, const PairDev* __restrict__ pairs,
                        const double* __restrict__ poses, int level, int32_t num, int32_t den,
                        uint8_t* __restrict__ selected) {
  __shared__ double pose_s[24];
  __shared__ double R[9], t[3];
  __shared__ const float4* A_s;
  __shared__ int64_t n_s;
  __shared__ MapLevelDev lv_s;
  __shared__ int dyadic_s;
  __shared__ float Rf[9], map_lo[4], map_hi[4];
  __shared__ const float* cbox_s;
  __shared__ MapLevelDev cv_s;
  __shared__ unsigned long long prog;  // hits << 32 | processed points
  __shared__ int decided;              // 0 open, 1 selected, 2 rejected
  const int tid = threadIdx.x;
  const int32_t p = blockIdx.x;
  const PairDev pd = pairs[p];
  if (tid < 24) {
    pose_s[tid] = __ldg(poses + 12 * (int64_t)(tid < 12 ? pd.pi : pd.pj) + (tid % 12));
  } else if (tid == 32) {
    const CloudDev* cd = clouds[pd.src];
    A_s = cd->A;
    cbox_s = cd->chunk_box;
    n_s = cd->n;
  } else if (tid == 64) {
    const MapDev* md = maps[pd.tgt];
    lv_s = md->lv[level];
    dyadic_s = md->dyadic;
    for (int j = 0; j < 4; ++j) {
      map_lo[j] = md->box_lo[j];
      map_hi[j] = md->box_hi[j];
    }
    cv_s = md->lv[GVOX_OVL_CULL_AT_LEVEL ? level : md->levels - 1];
  }
  __syncthreads();
  if (tid == 0) {
    double v[3];
    relative_pose_dev(pose_s, pose_s + 12, R, t, v);
    for (int j = 0; j < 9; ++j) Rf[j] = (float)R[j];
    prog = 0ull;
    decided = 0;
  }
  __syncthreads();
  const MapLevelDev lv = lv_s;
  const int dyadic = dyadic_s;
  const float4* __restrict__ A = A_s;
  const int64_t n = n_s;  // < 2^32 (cloud sizes are int32-indexed on the device)
  const float* cbox = cbox_s;
  const int64_t nchunks = (n + 31) >> 5;
  const int64_t need = (n * (int64_t)num) / den + 1;  // count * den > n * num <=> count >= need
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t msteps = (n + kThreads - 1) / kThreads;
  const uint32_t tail_pts = (uint32_t)(n - 32 * (nchunks - 1));  // points of the last chunk
  // points in the chunks of sub-steps mb + j, j in mask (all 32 but the tail chunk)
  auto mask_pts = [&](int64_t mb, uint32_t mask) -> uint32_t {
    uint32_t pts = 32u * (uint32_t)__popc(mask);
    const int64_t jt = (nchunks - 1 - warp) / (kThreads / 32) - mb;  // sub-step of the tail chunk
    if ((nchunks - 1 - warp) % (kThreads / 32) == 0 && jt >= 0 && jt < 32 && (mask >> jt & 1u))
      pts -= 32u - tail_pts;
    return pts;
  };
  // point m * kThreads + 32 warp + lane (sub-step m's chunk of this warp) exists
  // iff m < m_lim; its record sits a fixed stride from the lane's first one
  const int32_t m_lim = (int32_t)((n - 32 * warp - lane + kThreads - 1) / kThreads);
  const float4* __restrict__ A_lane = A + (warp * 96 + lane);
  auto probe = [&](int32_t m) -> int {
    if (m >= m_lim) return 0;
    const float4 a = __ldg(A_lane + m * (kThreads / 32 * 96));
    const double mx = a.x, my = a.y, mz = a.z;
    const double qx = __fma_rn(R[0], mx, __fma_rn(R[1], my, __fma_rn(R[2], mz, t[0])));
    const double qy = __fma_rn(R[3], mx, __fma_rn(R[4], my, __fma_rn(R[5], mz, t[1])));
    const double qz = __fma_rn(R[6], mx, __fma_rn(R[7], my, __fma_rn(R[8], mz, t[2])));
    const int32_t kx = voxel_coord0(qx, lv.r, lv.inv_r, DYADIC);
    const int32_t ky = voxel_coord0(qy, lv.r, lv.inv_r, DYADIC);
    const int32_t kz = voxel_coord0(qz, lv.r, lv.inv_r, DYADIC);
    return lookup_level<ALL_DENSE>(lv, kx, ky, kz) >= 0;
  };
  // publish (h, pts); true once the CTA's decision is certain
  auto publish = [&](int h, uint32_t pts) -> bool {
    int dec = 0;
    if (lane == 0) {
      const unsigned long long add = ((unsigned long long)(unsigned)h << 32) | pts;
      const unsigned long long now = atomicAdd(&prog, add) + add;
      const int64_t hits = (int64_t)(now >> 32), proc = (int64_t)(now & 0xffffffffull);
      if (hits >= need) dec = 1;
      else if (hits + (n - proc) < need) dec = 2;
      if (dec) atomicExch(&decided, dec);
      else dec = *((volatile int*)&decided);
    }
    return __shfl_sync(0xffffffffu, dec, 0) != 0;
  };
#pragma unroll 1
  for (int64_t mb = 0; mb < msteps; mb += 32) {
    uint32_t cull = 0;
    if (GVOX_OVL_CULL && cbox)
      cull = cull_ballot(cbox, mb * (kThreads / 32) + warp, kThreads / 32, nchunks, Rf, t, map_lo,
                         map_hi, (cv_s.dense && cv_s.grid) ? &cv_s : nullptr);
    // this warp's real chunks of the word (sub-steps whose chunk exists)
    uint32_t real = 0;
    {
      const int64_t c0 = mb * (kThreads / 32) + warp;  // chunk of sub-step mb
      const int64_t left = c0 < nchunks ? (nchunks - 1 - c0) / (kThreads / 32) + 1 : 0;
      real = left >= 32 ? 0xffffffffu : ((1u << left) - 1u);
    }
    uint32_t w = ~cull & real;
    const uint32_t culled = cull & real;
    bool stop = culled && publish(0, mask_pts(mb, culled));  // culled: processed, no hit
    while (w && !stop) {
      uint32_t g = 0;  // the group's chunks (up to four)
      int h;
      const int j0 = __ffs(w) - 1;
      w &= w - 1;
      g |= 1u << j0;
      if (w) {
        const int j1 = __ffs(w) - 1;
        w &= w - 1;
        g |= 1u << j1;
        if (w) {
          const int j2 = __ffs(w) - 1;
          w &= w - 1;
          g |= 1u << j2;
          if (w) {
            const int j3 = __ffs(w) - 1;
            w &= w - 1;
            g |= 1u << j3;
            h = (probe(mb + j0) + probe(mb + j1)) + (probe(mb + j2) + probe(mb + j3));
          } else {
            h = probe(mb + j0) + probe(mb + j1) + probe(mb + j2);
          }
        } else {
          h = probe(mb + j0) + probe(mb + j1);
        }
      } else {
        h = probe(mb + j0);
      }
      h = __reduce_add_sync(0xffffffffu, h);
      stop = publish(h, mask_pts(mb, g));
    }
    if (stop) break;
  }
  __syncthreads();
  if (tid == 0) {
    // undecided only if every point was processed without a certain decision
    // before the last publish (n = 0, or the final snapshot): decide on the count
    const int dec = decided;
    selected[p] = (dec == 1 || (dec == 0 && (int64_t)(prog >> 32) >= need)) ? 1 : 0;
  }
}

}  // namespace

void launch_overlap(const CloudDev* const* clouds, const MapDev* const* maps, const PairDev* pairs,
                    const int32_t* tile_start, int64_t num_pairs, int64_t num_tiles, int tile_pts,
                    const double* poses, int level, int32_t* tile_pair, int32_t* counts,
                    bool all_dense, cudaStream_t stream) {
  if (num_tiles <= 0) return;
  if (all_dense)
    k_overlap<true><<<(unsigned)num_tiles, kThreads, 0, stream>>>(
        clouds, maps, pairs, tile_start, tile_pair, tile_pts, poses, level, counts);
  else
    k_overlap<false><<<(unsigned)num_tiles, kThreads, 0, stream>>>(
        clouds, maps, pairs, tile_start, tile_pair, tile_pts, poses, level, counts);
  note_launch();
}

}  // namespace gvox

namespace gvox {
void launch_overlap_select(const CloudDev* const* clouds, const MapDev* const* maps,
                           const PairDev* pairs, int64_t num_pairs, const double* poses, int level,
                           int32_t num, int32_t den, uint8_t* selected, bool all_dense,
                           bool all_dyadic, cudaStream_t stream) {
  if (num_pairs <= 0) return;
  if (GVOX_OVL_NOBAR) {
    auto* k = all_dense ? (all_dyadic ? k_overlap_select_nb<true, true> : k_overlap_select_nb<true, false>)
                        : (all_dyadic ? k_overlap_select_nb<false, true> : k_overlap_select_nb<false, false>);
    k<<<(unsigned)num_pairs, kThreads, 0, stream>>>(clouds, maps, pairs, poses, level, num, den,
                                                    selected);
  } else if (all_dense)
    k_overlap_select<true><<<(unsigned)num_pairs, kThreads, 0, stream>>>(
        clouds, maps, pairs, poses, level, num, den, selected);
  else
    k_overlap_select<false><<<(unsigned)num_pairs, kThreads, 0, stream>>>(
        clouds, maps, pairs, poses, level, num, den, selected);
  note_launch();
}
}  // namespace gvox

// ------------------------------------------------------------ union overlap
namespace gvox {
namespace {

constexpr int kUnionChunk = 32;  // members staged in shared memory at a time

// P:280 keyframe insertion test: "the overlap rate between that frame and the
// union of all keyframes".  One CTA per tile of a query's source points; each
// thread owns up to 32 points (bit m of `hit`: point kb + m * 256 + tid) and
// tests them against the members in chunks of kUnionChunk (poses composed
// in fp64 with the pinned order, Q10), stopping at the first member whose
// voxel at `level` is occupied.  Integer counts: exact, order-independent.
__global__ void __launch_bounds__(kThreads)
    k_overlap_union(const CloudDev* const* __restrict__ clouds, const MapDev* const* __restrict__ maps,
                    const UnionQueryDev* __restrict__ queries, const UnionMemberDev* __restrict__ members,
                    const int32_t* __restrict__ tile_start, const int32_t* __restrict__ tile_query,
                    int tile_pts, const double* __restrict__ poses, int level,
                    int32_t* __restrict__ counts) {
  __shared__ double Rt_s[kUnionChunk][12];  // R (9), t (3) of T_j^-1 T_i
  __shared__ MapLevelDev lv_s[kUnionChunk];
  __shared__ int32_t dy_s[kUnionChunk];
  __shared__ int warp_cnt[kThreads / 32];
  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;
  const int32_t qi = __ldg(tile_query + tile);
  const UnionQueryDev q = queries[qi];
  const CloudDev* cd = clouds[q.src];
  const float4* __restrict__ A = cd->A;
  const int64_t kb = (int64_t)(tile - __ldg(tile_start + qi)) * tile_pts;
  const int64_t ke = kb + tile_pts < cd->n ? kb + tile_pts : cd->n;
  const int nm = (int)((ke - kb + kThreads - 1) / kThreads);  // <= 32
  const double* Ti = poses + 12 * (int64_t)q.pi;
  uint32_t hit = 0;
  for (int c0 = 0; c0 < q.count; c0 += kUnionChunk) {
    const int nc = q.count - c0 < kUnionChunk ? q.count - c0 : kUnionChunk;
    __syncthreads();  // previous chunk no longer in use
    if (tid < nc) {
      const UnionMemberDev mb = members[q.first + c0 + tid];
      const MapDev* md = maps[mb.tgt];
      double Tj[12], Tl[12], v[3];
      for (int j = 0; j < 12; ++j) {
        Tj[j] = __ldg(poses + 12 * (int64_t)mb.pj + j);
        Tl[j] = __ldg(Ti + j);
      }
      relative_pose_dev(Tl, Tj, Rt_s[tid], Rt_s[tid] + 9, v);
      lv_s[tid] = md->lv[level];
      dy_s[tid] = md->dyadic;
    }
    __syncthreads();
    for (int m = 0; m < nm; ++m) {
      if (hit >> m & 1u) continue;
      const int64_t k = kb + (int64_t)m * kThreads + tid;
      if (k >= ke) break;
      const float4 a = __ldg(A + pt_off(k));
      const double mx = a.x, my = a.y, mz = a.z;
      for (int j = 0; j < nc; ++j) {
        const double* R = Rt_s[j];
        const double qx = __fma_rn(R[0], mx, __fma_rn(R[1], my, __fma_rn(R[2], mz, R[9])));
        const double qy = __fma_rn(R[3], mx, __fma_rn(R[4], my, __fma_rn(R[5], mz, R[10])));
        const double qz = __fma_rn(R[6], mx, __fma_rn(R[7], my, __fma_rn(R[8], mz, R[11])));
        const MapLevelDev& lv = lv_s[j];
        const int32_t kx = voxel_coord0(qx, lv.r, lv.inv_r, dy_s[j]);
        const int32_t ky = voxel_coord0(qy, lv.r, lv.inv_r, dy_s[j]);
        const int32_t kz = voxel_coord0(qz, lv.r, lv.inv_r, dy_s[j]);
        if (lookup_level<false>(lv, kx, ky, kz) >= 0) {
          hit |= 1u << m;
          break;
        }
      }
    }
  }
  int cnt = __popc(hit);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((tid & 31) == 0) warp_cnt[tid >> 5] = cnt;
  __syncthreads();
  if (tid == 0) {
    int s = 0;
    for (int w = 0; w < kThreads / 32; ++w) s += warp_cnt[w];
    if (s) atomicAdd(counts + qi, s);
  }
}

}  // namespace

void launch_overlap_union(const CloudDev* const* clouds, const MapDev* const* maps,
                          const UnionQueryDev* queries, const UnionMemberDev* members,
                          const int32_t* tile_start, const int32_t* tile_query, int64_t num_tiles,
                          int tile_pts, const double* poses, int level, int32_t* counts,
                          cudaStream_t stream) {
  if (num_tiles <= 0) return;
  k_overlap_union<<<(unsigned)num_tiles, kThreads, 0, stream>>>(
      clouds, maps, queries, members, tile_start, tile_query, tile_pts, poses, level, counts);
  note_launch();
}

}  // namespace gvox
