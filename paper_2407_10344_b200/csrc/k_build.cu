// k_build.cu -- cloud packing, voxelmap build (K1) and lookup kernels.
//
// Voxelmap ("we create a sparse voxelmap with spatial voxel hashing and
// take the average of the points and their covariances in each voxel";
// multi-resolution r_l = r0 2^l).  B200 design:
//  phase 1  one thread per (point, level): fp64 key, open-addressing insert
//           with a 64-bit atomicCAS into a temporary per-(map, level) table;
//           the inserting thread takes a compact voxel index (atomicAdd).
//  -- host reads the voxel counts (one sync per chunk) and sizes the final
//     arrays exactly --
//  phase 2  one thread per (point, level): FIXED-POINT integer accumulation
//           (64-bit atomicAdd) of the mean offset within the voxel, the
//           covariance and the count.  Integer addition is associative, so
//           the result is bitwise independent of scheduling.
//  phase 3  one thread per voxel: mean/cov = sums / count, stored as fp32
//           offset-from-centre and fp32 covariance; insert into the final
//           table (capacity 2^k >= 2V).
#include <climits>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "k_common.cuh"

namespace gvox {

namespace {

__device__ inline bool finite3(float a, float b, float c) {
  return isfinite(a) && isfinite(b) && isfinite(c);
}

// Pack the cloud's points into the chunked layout (gvox_internal.h) and gather
// its statistics: flag (non-finite input), max |C_ij|, min / max of the means
// (order-preserving ints), and the per-32-point chunk boxes.  Every warp walks
// whole 32-point chunks, grid-strided (a warp packs many chunks, so its stores
// drain while it works on the next ones -- one point per thread left the warps
// waiting at exit for their stores, r02u: 26.8 ms for C5's 2e8 points), and
// keeps its statistics in registers: one set of atomics per warp at the end.
__device__ __forceinline__ void cloud_pack_body(const float* __restrict__ mu,
                                                const float* __restrict__ cov,
                                                const float* __restrict__ nrm, int64_t n,
                                                float4* __restrict__ P,
                                                float* __restrict__ chunk_box,
                                                int32_t* __restrict__ stats, int64_t warp0,
                                                int64_t nwarps) {
  const int lane = threadIdx.x & 31;
  float cm = 0.f;
  bool bad = false;
  int32_t lox = INT_MAX, loy = INT_MAX, loz = INT_MAX, hix = INT_MIN, hiy = INT_MIN, hiz = INT_MIN;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  for (int64_t ch = warp0; ch < nchunks; ch += nwarps) {
    const int64_t i = ch * kChunk + lane;
    const bool in = i < n;
    float x = 0.f, y = 0.f, z = 0.f;
    if (in) {
      x = mu[3 * i];
      y = mu[3 * i + 1];
      z = mu[3 * i + 2];
      const float c0 = cov[6 * i], c1 = cov[6 * i + 1], c2 = cov[6 * i + 2];
      const float c3 = cov[6 * i + 3], c4 = cov[6 * i + 4], c5 = cov[6 * i + 5];
      float nx = 0.f, ny = 0.f, nz = 0.f;
      if (nrm) {
        nx = nrm[3 * i];
        ny = nrm[3 * i + 1];
        nz = nrm[3 * i + 2];
      }
      const bool b = !(finite3(x, y, z) && finite3(c0, c1, c2) && finite3(c3, c4, c5) &&
                       finite3(nx, ny, nz));
      bad |= b;
      float4* r = P + pt_off(i);
      r[0] = make_float4(x, y, z, c0);
      r[32] = make_float4(c1, c2, c3, c4);
      r[64] = make_float4(c5, nx, ny, nz);
      if (!b) {
        cm = fmaxf(cm, fmaxf(fmaxf(fmaxf(fabsf(c0), fabsf(c1)), fmaxf(fabsf(c2), fabsf(c3))),
                             fmaxf(fabsf(c4), fabsf(c5))));
        const int32_t ox = float_to_ordered(x), oy = float_to_ordered(y), oz = float_to_ordered(z);
        lox = min(lox, ox); hix = max(hix, ox);
        loy = min(loy, oy); hiy = max(hiy, oy);
        loz = min(loz, oz); hiz = max(hiz, oz);
      }
    }
    // the chunk's box of means (points of the chunk only)
    float bl0 = in ? x : INFINITY, bl1 = in ? y : INFINITY, bl2 = in ? z : INFINITY;
    float bh0 = in ? x : -INFINITY, bh1 = in ? y : -INFINITY, bh2 = in ? z : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bl0 = fminf(bl0, __shfl_xor_sync(0xffffffffu, bl0, o));
      bl1 = fminf(bl1, __shfl_xor_sync(0xffffffffu, bl1, o));
      bl2 = fminf(bl2, __shfl_xor_sync(0xffffffffu, bl2, o));
      bh0 = fmaxf(bh0, __shfl_xor_sync(0xffffffffu, bh0, o));
      bh1 = fmaxf(bh1, __shfl_xor_sync(0xffffffffu, bh1, o));
      bh2 = fmaxf(bh2, __shfl_xor_sync(0xffffffffu, bh2, o));
    }
    if (lane < 6)
      chunk_box[6 * ch + lane] = lane == 0 ? bl0 : lane == 1 ? bl1 : lane == 2 ? bl2
                               : lane == 3 ? bh0 : lane == 4 ? bh1 : bh2;
  }
  // warp reductions of the statistics, then one atomic per warp and statistic
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    lox = min(lox, __shfl_xor_sync(0xffffffffu, lox, o));
    loy = min(loy, __shfl_xor_sync(0xffffffffu, loy, o));
    loz = min(loz, __shfl_xor_sync(0xffffffffu, loz, o));
    hix = max(hix, __shfl_xor_sync(0xffffffffu, hix, o));
    hiy = max(hiy, __shfl_xor_sync(0xffffffffu, hiy, o));
    hiz = max(hiz, __shfl_xor_sync(0xffffffffu, hiz, o));
  }
  const unsigned anybad = __ballot_sync(0xffffffffu, bad);
  if (lane == 0) {
    if (anybad) atomicOr(stats, 1);
    if (cm > 0.f) atomicMax(reinterpret_cast<uint32_t*>(stats + 1), __float_as_uint(cm));
    if (lox != INT_MAX) {
      atomicMin(stats + 2, lox);
      atomicMin(stats + 3, loy);
      atomicMin(stats + 4, loz);
      atomicMax(stats + 5, hix);
      atomicMax(stats + 6, hiy);
      atomicMax(stats + 7, hiz);
    }
  }
}

constexpr int kPackBlocksPerCloud = 16;  // 128 warps per cloud, grid-strided over its chunks

__global__ void k_cloud_pack(const float* __restrict__ mu, const float* __restrict__ cov,
                             const float* __restrict__ nrm, int64_t n, float4* __restrict__ P,
                             float* __restrict__ chunk_box, int32_t* __restrict__ stats) {
  cloud_pack_body(mu, cov, nrm, n, P, chunk_box, stats,
                  ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5,
                  ((int64_t)gridDim.x * blockDim.x) >> 5);
}

// All clouds of a batch in one launch: blockIdx.y = cloud.
__global__ void k_cloud_pack_batch(const PackSeg* __restrict__ segs) {
  const PackSeg sg = segs[blockIdx.y];
  cloud_pack_body(sg.mu, sg.cov, sg.nrm, sg.n, sg.P, sg.chunk_box, sg.stats,
                  ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5,
                  ((int64_t)gridDim.x * blockDim.x) >> 5);
}

// Both passes aggregate within a warp: lanes holding the same (map, key) --
// frequent, since consecutive points are spatially coherent -- are grouped with
// __match_any_sync and only the group leader touches the table / issues the
// atomics.  Every lane runs every level (inactive lanes carry unique dummy
// keys) so the warp stays converged for the *_sync collectives.

// Grids are 2D: blockIdx.y = segment (cloud), blockIdx.x * blockDim.x +
// threadIdx.x = point within it, so a block never straddles two maps.
#ifndef GVOX_INS_KNOWN_IDX
#define GVOX_INS_KNOWN_IDX 1
#endif
#ifndef GVOX_INS_SEG_MAJOR
#define GVOX_INS_SEG_MAJOR 0  // r02ak: build 15.30 vs 15.21 ms (off)
#endif
#ifndef GVOX_INS_MINB
#define GVOX_INS_MINB 8
#endif
#ifndef GVOX_ACC_MINB
#define GVOX_ACC_MINB 4
#endif
// accumulation: segmented run sums when a warp has more than this many groups
#ifndef GVOX_ACC_SEG_MIN
#define GVOX_ACC_SEG_MIN 1
#endif
// accumulation: level-independent covariance terms converted once per point
#ifndef GVOX_ACC_HOIST
#define GVOX_ACC_HOIST 1
#endif
// segmented sums: only as many doubling rounds as the warp's longest run
#ifndef GVOX_ACC_MAXRUN
#define GVOX_ACC_MAXRUN 1
#endif

// SEG_MAJOR: blockIdx.x = segment, blockIdx.y = block of the segment, so the
// CTAs resident at one time belong to many maps and their per-map voxel
// counters (one global atomicAdd per block and level) are not all contended
// by the same few maps' blocks
template <int kMaxL, bool SEG_MAJOR = false>
__global__ void __launch_bounds__(256, GVOX_INS_MINB) k_build_insert(const BuildSeg* __restrict__ segs, int levels, double r0,
                               double inv_r0, int dyadic, int32_t* __restrict__ pslot,
                               int32_t* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const unsigned bseg = SEG_MAJOR ? blockIdx.x : blockIdx.y, bblk = SEG_MAJOR ? blockIdx.y : blockIdx.x;
  const BuildSeg& sg = segs[bseg];
  const int64_t k = (int64_t)bblk * blockDim.x + threadIdx.x;
  const bool valid = k < sg.n;
  // (block-uniform exit only: the index allocation below uses block barriers)
  if ((int64_t)bblk * blockDim.x >= sg.n) return;
  int32_t k0x = 0, k0y = 0, k0z = 0;
  if (valid) {
    const float4 a = __ldg(sg.A + pt_off(k));
    k0x = voxel_coord0((double)a.x, r0, inv_r0, dyadic);
    k0y = voxel_coord0((double)a.y, r0, inv_r0, dyadic);
    k0z = voxel_coord0((double)a.z, r0, inv_r0, dyadic);
  }
  // 1) keys and warp groups of every level; 2) the group leaders' first CAS of
  // every level issued back to back (independent L2 round trips in flight
  // together); 3) collisions resolved by linear probing; 4) new voxels take
  // consecutive indices with one atomicAdd per warp and level.
  uint64_t key[kMaxL];
  uint64_t h[kMaxL];
  unsigned long long prev[kMaxL];
  int32_t dold[kMaxL];  // dense levels: the cell's value before the claim (an index >= 0: known)
  bool lead[kMaxL];
  int leader[kMaxL];
#pragma unroll
  for (int l = 0; l < kMaxL; ++l) {
    lead[l] = false;
    leader[l] = 0;
    if (l >= levels) continue;
    // floor(x / r_l) = floor(x / r0) >> l exactly (r_l = r0 2^l)
    const int32_t kx = k0x >> l, ky = k0y >> l, kz = k0z >> l;
    const bool inr = valid && key_in_range(kx) && key_in_range(ky) && key_in_range(kz);
    if (valid && !inr) atomicOr(err, 1);
    // real keys are < 2^63; dummies (~0 - lane) are distinct and never inserted
    key[l] = inr ? pack_key(kx, ky, kz) : ~0ull - (uint64_t)lane;
    const unsigned grp = __match_any_sync(0xffffffffu, key[l]);
    leader[l] = __ffs(grp) - 1;
    lead[l] = lane == leader[l] && inr;
  }
#pragma unroll
  for (int l = 0; l < kMaxL; ++l) {
    dold[l] = -1;
    if (lead[l]) {
      if (sg.box[l].dense) {
        // dense level: claim the final grid cell (-1 -> -2); h = cell
        const LevelBox& bx = sg.box[l];
        h[l] = (uint64_t)((uint32_t)((k0x >> l) - bx.x0) * bx.syz +
                          (uint32_t)((k0y >> l) - bx.y0) * bx.dz + (uint32_t)((k0z >> l) - bx.z0));
        const int old = atomicCAS(bx.grid + h[l], -1, -2);
        prev[l] = old == -1 ? kEmptyKey : key[l];  // "empty" = new voxel, else found
        dold[l] = old;
      } else {
        h[l] = hash_slot(key[l], sg.tmp_shift);
        prev[l] = atomicCAS(reinterpret_cast<unsigned long long*>(&sg.tmp_slots[l][h[l]].x),
                            kEmptyKey, key[l]);
      }
    }
  }
  // probing (hash levels only), then the index allocation aggregated over the
  // block: warp counts -> shared-memory offsets -> one global atomicAdd per
  // block and level (the per-map counters are the contended addresses)
  __shared__ int32_t blk_cnt[kMaxL], blk_base[kMaxL];
  bool is_new[kMaxL];
  int32_t h_out[kMaxL];
  unsigned new_mask[kMaxL];
  int32_t woff[kMaxL];
  if (threadIdx.x < kMaxL) blk_cnt[threadIdx.x] = 0;
  __syncthreads();
#pragma unroll
  for (int l = 0; l < kMaxL; ++l) {
    is_new[l] = false;
    h_out[l] = -1;
    new_mask[l] = 0;
    woff[l] = 0;
    if (l >= levels) continue;
    if (lead[l]) {
      while (prev[l] != kEmptyKey && prev[l] != key[l]) {
        h[l] = (h[l] + 1) & sg.tmp_mask;
        prev[l] = atomicCAS(reinterpret_cast<unsigned long long*>(&sg.tmp_slots[l][h[l]].x),
                            kEmptyKey, key[l]);
      }
      is_new[l] = prev[l] == kEmptyKey;
      h_out[l] = (int32_t)h[l];
    }
    new_mask[l] = __ballot_sync(0xffffffffu, is_new[l]);
    if (new_mask[l] && lane == __ffs(new_mask[l]) - 1)
      woff[l] = atomicAdd(&blk_cnt[l], __popc(new_mask[l]));
  }
  __syncthreads();
  if (threadIdx.x < levels && blk_cnt[threadIdx.x] > 0)
    blk_base[threadIdx.x] = atomicAdd(sg.counter + threadIdx.x, blk_cnt[threadIdx.x]);
  __syncthreads();
#pragma unroll
  for (int l = 0; l < kMaxL; ++l) {
    if (l >= levels) break;
    // the voxel index where this build already knows it: a new voxel's, or a
    // found dense cell that held an index (not a -2 claim still being filled)
    int32_t known = lead[l] && dold[l] >= 0 ? dold[l] : -1;
    if (new_mask[l]) {
      const int32_t b =
          blk_base[l] + __shfl_sync(0xffffffffu, woff[l], __ffs(new_mask[l]) - 1);
      if (is_new[l]) {
        const int32_t idx = b + __popc(new_mask[l] & ((1u << lane) - 1u));
        known = idx;
        if (sg.box[l].dense)
          sg.box[l].grid[h_out[l]] = idx;
        else
          sg.tmp_slots[l][h_out[l]].y = (unsigned long long)(uint32_t)idx | 0xFFFFFFFF00000000ull;
        sg.keys_by_idx[l][idx] = key[l];
        if (sg.acc) {  // sync-free build: this voxel's accumulators start at zero
          ulonglong2* a = reinterpret_cast<ulonglong2*>(sg.acc + (sg.acc_offset[l] + idx) * 10);
#pragma unroll
          for (int j = 0; j < 5; ++j) a[j] = make_ulonglong2(0ull, 0ull);
        }
      }
    }
    const int32_t hl = __shfl_sync(0xffffffffu, h_out[l], leader[l]);
    const int32_t kidx = __shfl_sync(0xffffffffu, known, leader[l]);
    const bool inr = key[l] < (1ull << 63);
    // (lifted builds accumulate only level 0 from the points).  Slot: the cell
    // / hash slot (>= 0, resolved by the accumulation), -1 no voxel, or -(index
    // + 2) for a dense level whose index is already known here -- the
    // accumulation then skips the grid read (one 32 B sector per point)
    if (valid && (!sg.lift || l == 0))
      pslot[sg.pl_offset + l * sg.pl_stride + k] =
          !inr ? -1 : (GVOX_INS_KNOWN_IDX && sg.box[l].dense && kidx >= 0) ? -(kidx + 2) : hl;
  }
}

__device__ inline unsigned long long to_fixed(double x) {
  return (unsigned long long)__double2ll_rn(x);
}

__global__ void __launch_bounds__(256, GVOX_ACC_MINB) k_build_accum(const BuildSeg* __restrict__ bsegs, const AccumSeg* __restrict__ segs,
                              int levels, double r0, double inv_r0, int dyadic,
                              const int32_t* __restrict__ pslot,
                              unsigned long long* __restrict__ acc) {
  const int lane = threadIdx.x & 31;
  const AccumSeg& sg = segs[blockIdx.y];
  const BuildSeg& bs = bsegs[blockIdx.y];
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = k < sg.n;
  if (__all_sync(0xffffffffu, !valid)) return;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a, c = a;
  if (valid) {
    const float4* r = sg.A + pt_off(k);
    a = __ldg(r);
    b = __ldg(r + 32);
    c = __ldg(r + 64);
  }
  const double x = a.x, y = a.y, z = a.z;
  const int32_t k0x = voxel_coord0(x, r0, inv_r0, dyadic);
  const int32_t k0y = voxel_coord0(y, r0, inv_r0, dyadic);
  const int32_t k0z = voxel_coord0(z, r0, inv_r0, dyadic);
  const float cv[6] = {a.w, b.x, b.y, b.z, b.w, c.x};
#if GVOX_ACC_HOIST
  // the covariance terms do not depend on the level: converted and split once.
  // (Lanes without a voxel need no zeroing: their index is unique to the lane,
  // so no run or group that is summed contains them.)
  unsigned cov_lo[6];
  int cov_hi[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    const unsigned long long f = to_fixed((double)cv[j] * sg.cov_scale);
    cov_lo[j] = (unsigned)(f & 0xFFFFFFull);
    cov_hi[j] = (int)((long long)f >> 24);
  }
#endif
  for (int l = 0; l < (bs.lift ? 1 : levels); ++l) {
    int32_t sl = valid ? pslot[sg.pl_offset + l * sg.pl_stride + k] : -1;
    const bool has = sl != -1;  // the point has a voxel at this level
    int32_t idx;
    if (bs.box[l].dense) {
      // dense level: the index the insert already knew (sl = -(idx + 2)), else
      // the final grid's (phase 1 is complete)
      idx = sl >= 0 ? __ldg(bs.box[l].grid + sl) : sl < -1 ? -sl - 2 : -1 - lane;
    } else {
      idx = sl >= 0 ? (int32_t)(uint32_t)bs.tmp_slots[l][sl].y : -1 - lane;
    }
    const unsigned grp = __match_any_sync(0xffffffffu, idx);
#if GVOX_ACC_HOIST
    unsigned lo_c[9];
    int hi_c[9];
    {
      const double r = ldexp(r0, l);
      const double S = sg.mu_scale[l];
      const unsigned long long o[3] = {to_fixed((x - (double)(k0x >> l) * r) * S),
                                       to_fixed((y - (double)(k0y >> l) * r) * S),
                                       to_fixed((z - (double)(k0z >> l) * r) * S)};
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        lo_c[j] = (unsigned)(o[j] & 0xFFFFFFull);
        hi_c[j] = (int)((long long)o[j] >> 24);
      }
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        lo_c[3 + j] = cov_lo[j];
        hi_c[3 + j] = cov_hi[j];
      }
    }
#else
    unsigned long long v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (has) {
      const double r = ldexp(r0, l);
      // offset of the point within its voxel (voxel corner = k_l * r_l), fixed point
      const double S = sg.mu_scale[l];
      v[0] = to_fixed((x - (double)(k0x >> l) * r) * S);
      v[1] = to_fixed((y - (double)(k0y >> l) * r) * S);
      v[2] = to_fixed((z - (double)(k0z >> l) * r) * S);
#pragma unroll
      for (int j = 0; j < 6; ++j) v[3 + j] = to_fixed((double)cv[j] * sg.cov_scale);
    }
    // group sums: one iteration per distinct group of the warp, each a set of
    // full-mask REDUX.SUM (uniform mask: the fast path) over two 32-bit chunks
    // of the fixed-point values (|v| < 2^46: low 24 bits unsigned, high part
    // signed; 32 lanes cannot overflow either chunk)
    unsigned lo_c[9];
    int hi_c[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      lo_c[j] = (unsigned)(v[j] & 0xFFFFFFull);
      hi_c[j] = (int)((long long)v[j] >> 24);
    }
#endif
    unsigned todo = __ballot_sync(0xffffffffu, has);
    // many groups (fine levels): segmented suffix sums over RUNS of equal index
    // in lane order (shuffles; cost independent of the group count), one set
    // of atomics per run head.  A voxel split over several runs gets several
    // atomic contributions -- integer sums, so the result is the same.
    const int ngroups = __popc(__ballot_sync(0xffffffffu, has && lane == __ffs(grp) - 1));
    if (ngroups > GVOX_ACC_SEG_MIN) {
      const int32_t idx_prev = __shfl_up_sync(0xffffffffu, idx, 1);
      const bool head = lane == 0 || idx != idx_prev;
      const unsigned H = __ballot_sync(0xffffffffu, head);
      const unsigned after = lane == 31 ? 0u : (H & (0xffffffffu << (lane + 1)));
      const int run_end = after ? __ffs(after) - 2 : 31;
      int cnt = has ? 1 : 0;
      // only as many doubling rounds as the warp's longest run needs
      const int max_run = GVOX_ACC_MAXRUN ? __reduce_max_sync(0xffffffffu, head ? (unsigned)(run_end - lane + 1) : 0u) : 32;
#pragma unroll 1
      for (int off = 1; off < max_run; off <<= 1) {
        const bool take = lane + off <= run_end;
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          const unsigned ol = __shfl_down_sync(0xffffffffu, lo_c[j], off);
          const int oh = __shfl_down_sync(0xffffffffu, hi_c[j], off);
          if (take) {
            lo_c[j] += ol;
            hi_c[j] += oh;
          }
        }
        const int oc = __shfl_down_sync(0xffffffffu, cnt, off);
        if (take) cnt += oc;
      }
      if (head && has) {
        unsigned long long* dst = acc + (sg.acc_offset[l] + idx) * 10;
#pragma unroll
        for (int j = 0; j < 9; ++j)
          atomicAdd(dst + j, (unsigned long long)((long long)hi_c[j] * (1ll << 24)) +
                                 (unsigned long long)lo_c[j]);
        atomicAdd(dst + 9, (unsigned long long)cnt);
      }
      continue;
    }
    while (todo) {
      const int ld = __ffs(todo) - 1;
      const unsigned g = __shfl_sync(0xffffffffu, grp, ld);
      const bool in = (g >> lane) & 1u;
      unsigned long long sum[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        const unsigned sl_ = __reduce_add_sync(0xffffffffu, in ? lo_c[j] : 0u);
        const int sh_ = __reduce_add_sync(0xffffffffu, in ? hi_c[j] : 0);
        sum[j] = (unsigned long long)((long long)sh_ * (1ll << 24)) + (unsigned long long)sl_;
      }
      if (lane == ld) {
        unsigned long long* dst = acc + (sg.acc_offset[l] + idx) * 10;
#pragma unroll
        for (int j = 0; j < 9; ++j) atomicAdd(dst + j, sum[j]);
        atomicAdd(dst + 9, (unsigned long long)__popc(g));
      }
      todo &= ~g;
    }
  }
}

#ifndef GVOX_FIN_MINB
#define GVOX_FIN_MINB 8
#endif
// Level l -> l + 1 of the accumulation (nested voxels: a level-(l+1) voxel is
// the union of the level-l voxels inside it).  The offsets are fixed
// point at ONE scale for every level (AccumSeg::mu_scale, 2^F / r_(L-1)), so a
// child's sums move to its parent's corner by adding count * (the child
// corner's offset in the parent) * scale, an exact integer (r_l * scale is a
// power of two); covariance sums and counts add as they are.  Integer sums:
// the parent's sums are bitwise those of summing its points directly.  One
// thread per level-l voxel, warp runs of equal parent summed by shuffles, one
// set of atomics per run.
__global__ void __launch_bounds__(256) k_build_lift(const BuildSeg* __restrict__ bsegs,
                                                    const AccumSeg* __restrict__ segs, int levels,
                                                    int l, double r0,
                                                    unsigned long long* __restrict__ acc) {
  const int lane = threadIdx.x & 31;
  const AccumSeg& sg = segs[blockIdx.y];
  const BuildSeg& bs = bsegs[blockIdx.y];
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nv = bs.counter[l];  // (final after the insert)
  if (__all_sync(0xffffffffu, v >= nv)) return;
  const bool valid = v < nv;
  unsigned long long val[10];
  int32_t pidx = -1 - lane;  // unique per lane unless a real parent is found
  if (valid) {
    const unsigned long long* src = acc + (sg.acc_offset[l] + v) * 10;
#pragma unroll
    for (int j = 0; j < 10; ++j) val[j] = src[j];
    const uint64_t key = bs.keys_by_idx[l][v];
    const int32_t kx = (int32_t)((key >> 42) & 0x1FFFFF) - kKeyHalf;
    const int32_t ky = (int32_t)((key >> 21) & 0x1FFFFF) - kKeyHalf;
    const int32_t kz = (int32_t)(key & 0x1FFFFF) - kKeyHalf;
    // the child corner's offset inside the parent, in fixed-point units
    const unsigned long long unit = (unsigned long long)(ldexp(r0, l) * sg.mu_scale[l]);
    const unsigned long long cnt = val[9];
    val[0] += cnt * unit * (unsigned long long)(kx & 1);
    val[1] += cnt * unit * (unsigned long long)(ky & 1);
    val[2] += cnt * unit * (unsigned long long)(kz & 1);
    const int32_t px = kx >> 1, py = ky >> 1, pz = kz >> 1;
    const LevelBox& bx = bs.box[l + 1];
    if (bx.dense) {
      pidx = bx.grid[(size_t)((uint32_t)(px - bx.x0) * bx.syz + (uint32_t)(py - bx.y0) * bx.dz +
                              (uint32_t)(pz - bx.z0))];
    } else {
      const uint64_t pk = pack_key(px, py, pz);
      uint64_t h = hash_slot(pk, bs.tmp_shift);
      for (;;) {
        const ulonglong2 e = bs.tmp_slots[l + 1][h];
        if (e.x == pk) {
          pidx = (int32_t)(uint32_t)e.y;
          break;
        }
        h = (h + 1) & bs.tmp_mask;  // (the parent exists: its points are the child's)
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 10; ++j) val[j] = 0ull;
  }
  // runs of equal parent in lane order; suffix sums by doubling (64-bit values)
  const int32_t prev = __shfl_up_sync(0xffffffffu, pidx, 1);
  const bool head = lane == 0 || pidx != prev;
  const unsigned H = __ballot_sync(0xffffffffu, head);
  const unsigned after = lane == 31 ? 0u : (H & (0xffffffffu << (lane + 1)));
  const int run_end = after ? __ffs(after) - 2 : 31;
  const int max_run = __reduce_max_sync(0xffffffffu, head ? (unsigned)(run_end - lane + 1) : 0u);
#pragma unroll 1
  for (int off = 1; off < max_run; off <<= 1) {
    const bool take = lane + off <= run_end;
#pragma unroll
    for (int j = 0; j < 10; ++j) {
      const unsigned long long o = __shfl_down_sync(0xffffffffu, val[j], off);
      if (take) val[j] += o;
    }
  }
  if (head && valid) {
    unsigned long long* dst = acc + (sg.acc_offset[l + 1] + pidx) * 10;
#pragma unroll
    for (int j = 0; j < 10; ++j) atomicAdd(dst + j, val[j]);
  }
  (void)levels;
}

__global__ void __launch_bounds__(256, GVOX_FIN_MINB) k_build_finalize(const FinalSeg* __restrict__ segs,
                                 const unsigned long long* __restrict__ acc) {
  const FinalSeg& sg = segs[blockIdx.y];  // one (segment, level) per grid row
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // record -1 of every level: all zeros, the record a lookup miss (index -1)
  // gathers in the linearize kernel's unconditional loads
  if (v < 3) sg.vox[v - 3] = make_float4(0.f, 0.f, 0.f, 0.f);
  const int32_t nv = *sg.nvox;
  if (v == 0 && sg.nvox_out) *sg.nvox_out = nv;  // the map keeps its count (no separate copy)
  if (v >= nv) return;
  const unsigned long long* src = acc + (sg.acc_offset + v) * 10;
  double cnt = (double)(long long)src[9];
  double inv = 1.0 / cnt;
  double m[3], cv[6];
  for (int j = 0; j < 3; ++j) m[j] = (double)(long long)src[j] * inv / sg.mu_scale - 0.5 * sg.r;
  for (int j = 0; j < 6; ++j) cv[j] = (double)(long long)src[3 + j] * inv / sg.cov_scale;
  float4* o = sg.vox + 3 * v;
  o[0] = make_float4((float)m[0], (float)m[1], (float)m[2], (float)cv[0]);
  // record layout {C.xy, C.yy, C.xz, C.yz}: pairs (xy, yy), (xz, yz) match the
  // packed-fp32 column pairs of R C R^T in the linearize kernel
  o[1] = make_float4((float)cv[1], (float)cv[3], (float)cv[2], (float)cv[4]);
  o[2] = make_float4((float)cv[5], __int_as_float((int)src[9]), 0.f, 0.f);
  uint64_t key = sg.keys_by_idx[v];
  sg.keys_out[v] = key;
  if (sg.grid) {
    const int32_t kx = (int32_t)((key >> 42) & 0x1FFFFF) - kKeyHalf;
    const int32_t ky = (int32_t)((key >> 21) & 0x1FFFFF) - kKeyHalf;
    const int32_t kz = (int32_t)(key & 0x1FFFFF) - kKeyHalf;
    sg.grid[((size_t)(kx - sg.x0) * sg.dy + (ky - sg.y0)) * sg.dz + (kz - sg.z0)] = (int32_t)v;
  }
  if (!sg.slots) return;
  uint64_t h = hash_slot(key, sg.shift);
  for (;;) {
    unsigned long long* kp = reinterpret_cast<unsigned long long*>(&sg.slots[h].x);
    unsigned long long prev = atomicCAS(kp, kEmptyKey, key);
    if (prev == kEmptyKey) {
      sg.slots[h].y = (unsigned long long)(uint32_t)v | 0xFFFFFFFF00000000ull;
      break;
    }
    h = (h + 1) & sg.mask;
  }
}

// One (map, level) per grid row: cell of voxel v back to -1 (empty).
__global__ void k_grid_reset(const ResetSeg* __restrict__ segs) {
  const ResetSeg& sg = segs[blockIdx.y];
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (!sg.nvox || v >= *sg.nvox) return;
  const uint64_t key = sg.keys[v];
  const int32_t kx = (int32_t)((key >> 42) & 0x1FFFFF) - kKeyHalf;
  const int32_t ky = (int32_t)((key >> 21) & 0x1FFFFF) - kKeyHalf;
  const int32_t kz = (int32_t)(key & 0x1FFFFF) - kKeyHalf;
  sg.grid[((size_t)(kx - sg.x0) * sg.dy + (ky - sg.y0)) * sg.dz + (kz - sg.z0)] = -1;
}

// Host -> device copy by the SMs: reads pinned (mapped) host memory over PCIe
// directly (ld.global.cv: the staging slots are rewritten by the host between
// uses, nothing may be cached), so the calls' small input blocks never queue on
// the copy engines behind a bulk upload running on another stream.
__global__ void k_h2d_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, int64_t bytes) {
  const int64_t n16 = bytes >> 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  if (aligned) {
    for (int64_t i = t0; i < n16; i += stride)
      reinterpret_cast<int4*>(dst)[i] = __ldcv(reinterpret_cast<const int4*>(src) + i);
    for (int64_t i = (n16 << 4) + t0; i < bytes; i += stride) dst[i] = *(const volatile uint8_t*)(src + i);
  } else {
    for (int64_t i = t0; i < bytes; i += stride) dst[i] = *(const volatile uint8_t*)(src + i);
  }
}

// Small blocks ride in the launch itself: the bytes are copied into the
// kernel's parameter buffer when the launch is enqueued (up to 32,000 bytes;
// the launch limit is 32,764) and the kernel stores them from the constant bank -- no PCIe
// round trip at execution time (k_h2d_copy's uncached loads of the pinned slot
// cost ~1-2 us each on the critical path of an odometry-sized call).
template <int N>
struct ParamBlock {
  int4 w[N / 16];
};
// up to 4 segments whose bytes ride in the parameter buffer (src = offset into
// the block) or are zero-filled (bytes < 0: -bytes zeros); blockIdx.y = segment
struct ParamSeg {
  void* dst;
  int32_t off, bytes;
};
template <int N>
struct ParamSegs {
  ParamSeg s[4];
  int4 w[N / 16];
};
template <int N>
__global__ void k_param_segments(const __grid_constant__ ParamSegs<N> p) {
  const ParamSeg sg = p.s[blockIdx.y];
  uint8_t* dst = static_cast<uint8_t*>(sg.dst);
  const bool zero = sg.bytes < 0;
  const int bytes = zero ? -sg.bytes : sg.bytes;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(p.w) + sg.off;
  const int n16 = bytes >> 4;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  if (((reinterpret_cast<uintptr_t>(dst) | (uintptr_t)sg.off) & 15) == 0) {
    for (int i = t0; i < n16; i += stride)
      reinterpret_cast<int4*>(dst)[i] = zero ? make_int4(0, 0, 0, 0) : reinterpret_cast<const int4*>(src)[i];
    for (int i = (n16 << 4) + t0; i < bytes; i += stride) dst[i] = zero ? 0 : src[i];
  } else {
    for (int i = t0; i < bytes; i += stride) dst[i] = zero ? 0 : src[i];
  }
}

template <int N>
__global__ void k_param_copy(const __grid_constant__ ParamBlock<N> p, uint8_t* __restrict__ dst,
                             int bytes) {
  const int n16 = bytes >> 4;
  const uint8_t* src = reinterpret_cast<const uint8_t*>(p.w);
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    for (int i = threadIdx.x; i < n16; i += blockDim.x) reinterpret_cast<int4*>(dst)[i] = p.w[i];
    for (int i = (n16 << 4) + threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
  } else {
    for (int i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
  }
}

// H2D segments (launch_h2d_segments): blockIdx.y = segment
struct H2DSegs {
  H2DSeg s[4];
};
__global__ void k_h2d_segments(const __grid_constant__ H2DSegs segs) {
  const H2DSeg sg = segs.s[blockIdx.y];
  uint8_t* dst = static_cast<uint8_t*>(sg.dst);
  const uint8_t* src = static_cast<const uint8_t*>(sg.src);
  const int64_t n16 = sg.bytes >> 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  if (src == nullptr) {
    if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      for (int64_t i = t0; i < n16; i += stride) reinterpret_cast<int4*>(dst)[i] = make_int4(0, 0, 0, 0);
      for (int64_t i = (n16 << 4) + t0; i < sg.bytes; i += stride) dst[i] = 0;
    } else {
      for (int64_t i = t0; i < sg.bytes; i += stride) dst[i] = 0;
    }
  } else if (aligned) {
    for (int64_t i = t0; i < n16; i += stride)
      reinterpret_cast<int4*>(dst)[i] = __ldcv(reinterpret_cast<const int4*>(src) + i);
    for (int64_t i = (n16 << 4) + t0; i < sg.bytes; i += stride) dst[i] = *(const volatile uint8_t*)(src + i);
  } else {
    for (int64_t i = t0; i < sg.bytes; i += stride) dst[i] = *(const volatile uint8_t*)(src + i);
  }
}

__global__ void k_fill_u64(uint64_t* p, uint64_t value, int64_t count) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < count; i += stride) p[i] = value;
}

__global__ void k_lookup(const MapDev* __restrict__ map, int level, const double* __restrict__ q,
                         int64_t n, int64_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const MapLevelDev& lv = map->lv[level];
  int dy = map->dyadic;
  int32_t kx = clamp_coord(voxel_coord0(q[3 * i], lv.r, lv.inv_r, dy));
  int32_t ky = clamp_coord(voxel_coord0(q[3 * i + 1], lv.r, lv.inv_r, dy));
  int32_t kz = clamp_coord(voxel_coord0(q[3 * i + 2], lv.r, lv.inv_r, dy));
  int64_t res = -1;
  if (lookup_level(lv, kx, ky, kz) >= 0) res = (int64_t)pack_key(kx, ky, kz);
  out[i] = res;
}

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

}  // namespace

void launch_cloud_pack(const float* mu, const float* cov, const float* nrm, int64_t n, float4* P,
                       float* chunk_box, int32_t* stats, cudaStream_t stream) {
  if (n <= 0) return;
  const unsigned blocks = std::min<unsigned>(grid_for(n, 256), 148 * 8);  // grid-strided chunks
  k_cloud_pack<<<blocks, 256, 0, stream>>>(mu, cov, nrm, n, P, chunk_box, stats);
  note_launch();
}

void launch_cloud_pack_batch(const PackSeg* segs_dev, int64_t count, int64_t max_n,
                             cudaStream_t stream) {
  if (count <= 0 || max_n <= 0) return;
  // (a batch of many clouds fills the GPU with a few blocks per cloud; one or a
  // few clouds get up to ~1200 blocks in all)
  const unsigned per_cloud = std::max<unsigned>(
      kPackBlocksPerCloud, (unsigned)std::min<int64_t>(148 * 8 / count, grid_for(max_n, 256)));
  dim3 grid(std::min<unsigned>(grid_for(max_n, 256), per_cloud), (unsigned)count);
  k_cloud_pack_batch<<<grid, 256, 0, stream>>>(segs_dev);
  note_launch();
}

void launch_build_insert(const BuildSeg* segs_dev, int64_t num_segs, int64_t max_seg_points,
                         int levels, double r0, int dyadic, int32_t* pslot, int32_t* err,
                         cudaStream_t stream) {
  if (num_segs <= 0 || max_seg_points <= 0) return;
  dim3 grid(grid_for(max_seg_points, 256), (unsigned)num_segs);
  const bool seg_major = GVOX_INS_SEG_MAJOR && num_segs > 1 && grid.x <= 65535;
  if (levels <= 3 && seg_major)
    k_build_insert<3, true><<<dim3(grid.y, grid.x), 256, 0, stream>>>(segs_dev, levels, r0, 1.0 / r0,
                                                                      dyadic, pslot, err);
  else if (levels <= 3)
    k_build_insert<3><<<grid, 256, 0, stream>>>(segs_dev, levels, r0, 1.0 / r0, dyadic, pslot, err);
  else
    k_build_insert<GVOX_MAX_LEVELS><<<grid, 256, 0, stream>>>(segs_dev, levels, r0, 1.0 / r0,
                                                              dyadic, pslot, err);
  note_launch();
}

void launch_build_accum(const BuildSeg* bsegs_dev, const AccumSeg* segs_dev, int64_t num_segs,
                        int64_t max_seg_points, int levels, double r0, int dyadic,
                        const int32_t* pslot, unsigned long long* acc, cudaStream_t stream) {
  if (num_segs <= 0 || max_seg_points <= 0) return;
  dim3 grid(grid_for(max_seg_points, 256), (unsigned)num_segs);
  k_build_accum<<<grid, 256, 0, stream>>>(bsegs_dev, segs_dev, levels, r0, 1.0 / r0, dyadic, pslot,
                                          acc);
  note_launch();
}

void launch_build_lift(const BuildSeg* bsegs_dev, const AccumSeg* segs_dev, int64_t num_segs,
                       int levels, const int64_t* max_level_voxels, double r0,
                       unsigned long long* acc, cudaStream_t stream) {
  if (num_segs <= 0) return;
  for (int l = 0; l + 1 < levels; ++l) {
    if (max_level_voxels[l] <= 0) continue;
    dim3 grid(grid_for(max_level_voxels[l], 256), (unsigned)num_segs);
    k_build_lift<<<grid, 256, 0, stream>>>(bsegs_dev, segs_dev, levels, l, r0, acc);
    note_launch();
  }
}

void launch_build_finalize(const FinalSeg* segs_dev, int64_t num_segs, int64_t max_seg_voxels,
                           const unsigned long long* acc, cudaStream_t stream) {
  if (num_segs <= 0) return;  // (runs for empty maps too: it writes the sentinel records)
  dim3 grid(grid_for(max_seg_voxels > 0 ? max_seg_voxels : 1, 256), (unsigned)num_segs);
  k_build_finalize<<<grid, 256, 0, stream>>>(segs_dev, acc);
  note_launch();
}

void launch_grid_reset(const ResetSeg* segs_dev, int64_t num_segs, int64_t max_seg_voxels,
                       cudaStream_t stream) {
  if (num_segs <= 0 || max_seg_voxels <= 0) return;
  dim3 grid(grid_for(max_seg_voxels, 256), (unsigned)num_segs);
  k_grid_reset<<<grid, 256, 0, stream>>>(segs_dev);
  note_launch();
}

// Calls' input blocks of up to GVOX_H2D_PARAM bytes (default 4096, at most
// 31,744) ride in the launch's parameter buffer.  With a bulk upload sharing
// PCIe (the pipelined e2e) the SM-driven copies' PCIe reads queue behind it
// while parameter bytes do not (r02av, the linearize block as parameters: C2
// e2e 0.423 -> 0.362-0.375 ms, C3 0.893 -> 0.801-0.807 ms, steps unchanged);
// but a large parameter buffer costs the host more than it saves the device
// on the host-bound small steps (r02aw, every block up to 31,744 B, i.e. also
// the ~22 KB build block: C2 step 0.1255 -> 0.133-0.137 ms, C1 0.097 ->
// 0.109 ms), so only blocks up to 4 KB go this way.  0: always SM-driven.
int64_t h2d_param_max() {
  static const int64_t v = [] {
    const char* e = std::getenv("GVOX_H2D_PARAM");
    return e ? std::min<int64_t>(std::max<int64_t>(std::atoll(e), 0), 31744) : (int64_t)4096;
  }();
  return v;
}

void launch_h2d_copy(void* dst, const void* pinned_src, int64_t bytes, cudaStream_t stream) {
  if (bytes <= 0) return;
  const int64_t param_max = h2d_param_max();
  if (bytes <= param_max) {
    auto go = [&](auto tag) {
      constexpr int N = decltype(tag)::value;
      ParamBlock<N> pb;
      std::memcpy(&pb, pinned_src, (size_t)bytes);
      k_param_copy<N><<<1, 256, 0, stream>>>(pb, (uint8_t*)dst, (int)bytes);
    };
    if (bytes <= 1024)
      go(std::integral_constant<int, 1024>{});
    else if (bytes <= 4096)
      go(std::integral_constant<int, 4096>{});
    else if (bytes <= 16384)
      go(std::integral_constant<int, 16384>{});
    else
      go(std::integral_constant<int, 31744>{});
    note_launch();
    return;
  }
  int64_t blocks = ((bytes >> 4) + 255) / 256;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 4));
  k_h2d_copy<<<(unsigned)blocks, 256, 0, stream>>>((uint8_t*)dst, (const uint8_t*)pinned_src, bytes);
  note_launch();
}

void launch_h2d_segments(const H2DSeg* segs, int n, cudaStream_t stream) {
  if (n <= 0) return;
  n = std::min(n, 4);
  {
    // every copied segment's bytes in the parameter buffer (16-byte aligned
    // offsets), zero-fills as negative sizes
    int64_t tot = 0;
    bool ok = true;
    for (int i = 0; i < n; ++i) {
      if (segs[i].bytes > INT32_MAX / 2) ok = false;
      if (segs[i].src) tot += (segs[i].bytes + 15) & ~int64_t(15);
    }
    if (ok && tot <= h2d_param_max()) {
      auto go = [&](auto tag) {
        constexpr int N = decltype(tag)::value;
        ParamSegs<N> pb;
        int32_t off = 0;
        for (int i = 0; i < n; ++i) {
          pb.s[i].dst = segs[i].dst;
          pb.s[i].off = off;
          if (segs[i].src) {
            std::memcpy(reinterpret_cast<char*>(pb.w) + off, segs[i].src, (size_t)segs[i].bytes);
            pb.s[i].bytes = (int32_t)segs[i].bytes;
            off += (int32_t)((segs[i].bytes + 15) & ~int64_t(15));
          } else {
            pb.s[i].bytes = -(int32_t)segs[i].bytes;
          }
        }
        int64_t mx = 0;
        for (int i = 0; i < n; ++i) mx = std::max<int64_t>(mx, segs[i].bytes);
        const unsigned bx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(((mx >> 4) + 255) / 256, 148 * 4));
        k_param_segments<N><<<dim3(bx, (unsigned)n), 256, 0, stream>>>(pb);
      };
      if (tot <= 1024)
        go(std::integral_constant<int, 1024>{});
      else if (tot <= 4096)
        go(std::integral_constant<int, 4096>{});
      else if (tot <= 16384)
        go(std::integral_constant<int, 16384>{});
      else
        go(std::integral_constant<int, 31744>{});
      note_launch();
      return;
    }
  }
  H2DSegs p{};
  int64_t mx = 0;
  for (int i = 0; i < n && i < 4; ++i) {
    p.s[i] = segs[i];
    mx = std::max<int64_t>(mx, segs[i].bytes);
  }
  if (mx <= 0) return;
  int64_t blocks = ((mx >> 4) + 255) / 256;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 4));
  k_h2d_segments<<<dim3((unsigned)blocks, (unsigned)std::min(n, 4)), 256, 0, stream>>>(p);
  note_launch();
}

void launch_fill_u64(uint64_t* p, uint64_t value, int64_t count, cudaStream_t stream) {
  if (count <= 0) return;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_fill_u64<<<(unsigned)blocks, 256, 0, stream>>>(p, value, count);
  note_launch();
}

void launch_lookup(const MapDev* map, int level, const double* q, int64_t n, int64_t* out,
                   cudaStream_t stream) {
  if (n <= 0) return;
  k_lookup<<<grid_for(n, 256), 256, 0, stream>>>(map, level, q, n, out);
  note_launch();
}

}  // namespace gvox
