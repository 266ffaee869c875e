// k_common.cuh -- device helpers shared by the gvox kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "gvox_internal.h"

namespace gvox {

// T_ij = T_j^-1 T_i and v = T_i^-1 t_j (reading Q1), with the pinned fma order
// of reading Q10: R_ij[a][b] = fma(Rj[0][a], Ri[0][b], fma(Rj[1][a], Ri[1][b],
// Rj[2][a] * Ri[2][b])); t_ij = R_j^T (t_i - t_j); v = R_i^T (t_j - t_i).
// Poses are row-major 3x4.
__device__ inline void relative_pose_dev(const double* Ti, const double* Tj, double* R, double* t,
                                         double* v) {
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      R[a * 3 + b] = __fma_rn(Tj[0 * 4 + a], Ti[0 * 4 + b],
                              __fma_rn(Tj[1 * 4 + a], Ti[1 * 4 + b],
                                       __dmul_rn(Tj[2 * 4 + a], Ti[2 * 4 + b])));
  double dt0 = __dsub_rn(Ti[3], Tj[3]), dt1 = __dsub_rn(Ti[7], Tj[7]), dt2 = __dsub_rn(Ti[11], Tj[11]);
#pragma unroll
  for (int a = 0; a < 3; ++a)
    t[a] = __fma_rn(Tj[0 * 4 + a], dt0, __fma_rn(Tj[1 * 4 + a], dt1, __dmul_rn(Tj[2 * 4 + a], dt2)));
  double dv0 = __dsub_rn(Tj[3], Ti[3]), dv1 = __dsub_rn(Tj[7], Ti[7]), dv2 = __dsub_rn(Tj[11], Ti[11]);
#pragma unroll
  for (int a = 0; a < 3; ++a)
    v[a] = __fma_rn(Ti[0 * 4 + a], dv0, __fma_rn(Ti[1 * 4 + a], dv1, __dmul_rn(Ti[2 * 4 + a], dv2)));
}

// floor(x / r) as int32, saturating (|result| >= 2^30 is out of key range at
// every level l <= 7).  For a power-of-two r the product by 1/r is exact and
// equals the correctly rounded quotient; otherwise an IEEE division is used.
__device__ inline int32_t voxel_coord0(double x, double r, double inv_r, int dyadic) {
  double s = dyadic ? __dmul_rn(x, inv_r) : __ddiv_rn(x, r);
  return __double2int_rd(s);
}

// Probe a level's hash table: voxel index or -1.
__device__ inline int32_t probe_hash(const MapLevelDev& lv, uint64_t key) {
  uint64_t h = hash_slot(key, lv.shift);
  for (;;) {
    ulonglong2 s = __ldg(lv.slots + h);
    if (s.x == key) return (int32_t)(uint32_t)s.y;
    if (s.x == kEmptyKey) return -1;
    h = (h + 1) & lv.mask;
  }
}

// Voxel index of level key (kx, ky, kz) or -1.  Keys must come from
// clamp_coord() so that the subtractions below cannot overflow.
template <bool ALL_DENSE = false>
__device__ inline int32_t lookup_level(const MapLevelDev& lv, int32_t kx, int32_t ky, int32_t kz) {
  if (ALL_DENSE || lv.dense) {
    const int4 b0 = *reinterpret_cast<const int4*>(&lv.x0);    // x0 y0 z0 dx
    const uint4 b1 = *reinterpret_cast<const uint4*>(&lv.dy);  // dy dz syz dense
    const uint32_t cx = (uint32_t)(kx - b0.x), cy = (uint32_t)(ky - b0.y), cz = (uint32_t)(kz - b0.z);
    if (cx >= (uint32_t)b0.w || cy >= b1.x || cz >= b1.y) return -1;
    return __ldg(lv.grid + (cx * b1.z + cy * b1.y + cz));  // < 2^31 cells: 32-bit index
  }
  if (!key_in_range(kx) || !key_in_range(ky) || !key_in_range(kz)) return -1;
  return probe_hash(lv, pack_key(kx, ky, kz));
}

// floor(x / r0) clamped to [-2^30, 2^30]: anything clamped is out of key range
// at every level l <= 7, and (k >> l) - x0 stays inside int32.
__device__ inline int32_t clamp_coord(int32_t k) {
  return min(max(k, -(1 << 30)), 1 << 30);
}

// Exact culling: true if no point of the source chunk (box lo/hi in the source
// frame) can fall inside the map's conservative box after q = R mu + t.
// Interval arithmetic in fp32 plus a 1 mm margin (far above its rounding).
__device__ inline bool chunk_culled(const float* box, const float* Rf, const double* t,
                                    const float* map_lo, const float* map_hi) {
  const float cx = 0.5f * (box[0] + box[3]), cy = 0.5f * (box[1] + box[4]), cz = 0.5f * (box[2] + box[5]);
  const float hx = 0.5f * (box[3] - box[0]), hy = 0.5f * (box[4] - box[1]), hz = 0.5f * (box[5] - box[2]);
  bool out = false;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float qc = fmaf(Rf[3 * a], cx, fmaf(Rf[3 * a + 1], cy, fmaf(Rf[3 * a + 2], cz, (float)t[a])));
    // half-extent of the rotated box, plus 1 mm and a relative term bounding the
    // fp32 rounding of Rf, t and the products (|terms| summed, not |qc|)
    const float mag = fabsf(Rf[3 * a]) * fabsf(cx) + fabsf(Rf[3 * a + 1]) * fabsf(cy) +
                      fabsf(Rf[3 * a + 2]) * fabsf(cz) + fabsf((float)t[a]);
    const float qh = fabsf(Rf[3 * a]) * hx + fabsf(Rf[3 * a + 1]) * hy + fabsf(Rf[3 * a + 2]) * hz +
                     1e-3f + 1e-6f * (mag + hx + hy + hz);
    out |= (qc + qh < map_lo[a]) || (qc - qh > map_hi[a]);
  }
  return out;
}

// culling loads row by row with an early exit (1), or all <= 27 at once (0).
// Measured (r02ag, full C5): linearize 121.9 vs 122.1 ms, screening 12.54 vs
// 12.89 ms -- most ranges are one or two rows and a live chunk usually exits at
// the first, so the predicated loads cost more than the saved round trips
#ifndef GVOX_CULL_ROWS
#define GVOX_CULL_ROWS 1
#endif

// Exact culling against the occupancy of a map's COARSEST level (dense grid):
// levels nest (a level-l voxel holding a map point lies inside that point's
// coarsest-level voxel), so a source point can hit a voxel at any level only if
// its coarsest-level cell is occupied.  The chunk's transformed box (fp32
// interval arithmetic, margins as chunk_culled) is mapped to a cell range; the
// chunk is culled if the range misses the grid or every cell in it is empty.
// Ranges wider than 3 cells on an axis, or coordinates beyond 2^22 cells, are
// not culled.
__device__ inline bool chunk_culled_grid(const float* box, const float* Rf, const double* t,
                                         const MapLevelDev& cv) {
  const float cx = 0.5f * (box[0] + box[3]), cy = 0.5f * (box[1] + box[4]), cz = 0.5f * (box[2] + box[5]);
  const float hx = 0.5f * (box[3] - box[0]), hy = 0.5f * (box[4] - box[1]), hz = 0.5f * (box[5] - box[2]);
  const float inv = (float)cv.inv_r;
  const int32_t org[3] = {cv.x0, cv.y0, cv.z0};
  const uint32_t dim[3] = {cv.dx, cv.dy, cv.dz};
  int32_t c0[3], nc[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float qc = fmaf(Rf[3 * a], cx, fmaf(Rf[3 * a + 1], cy, fmaf(Rf[3 * a + 2], cz, (float)t[a])));
    const float mag = fabsf(Rf[3 * a]) * fabsf(cx) + fabsf(Rf[3 * a + 1]) * fabsf(cy) +
                      fabsf(Rf[3 * a + 2]) * fabsf(cz) + fabsf((float)t[a]);
    const float qh = fabsf(Rf[3 * a]) * hx + fabsf(Rf[3 * a + 1]) * hy + fabsf(Rf[3 * a + 2]) * hz +
                     1e-3f + 1e-6f * (mag + hx + hy + hz);
    const float vlo = (qc - qh) * inv, vhi = (qc + qh) * inv;
    const float flo = floorf(vlo - (1e-5f * fabsf(vlo) + 1e-3f));
    const float fhi = floorf(vhi + (1e-5f * fabsf(vhi) + 1e-3f));
    if (!(fabsf(flo) < 4194304.f && fabsf(fhi) < 4194304.f)) return false;  // also NaN
    const int32_t lo = max((int32_t)flo - org[a], 0);
    const int32_t hi = min((int32_t)fhi - org[a], (int32_t)dim[a] - 1);
    if (lo > hi) return true;  // the range misses the grid: every cell empty
    c0[a] = lo;
    nc[a] = hi - lo + 1;
  }
  if (nc[0] > 3 || nc[1] > 3 || nc[2] > 3) return false;
#if GVOX_CULL_ROWS
  // up to 3 x 3 x 3 cells: one row of <= 3 cells along z per step, its loads
  // in flight together
  for (int i = 0; i < nc[0]; ++i)
    for (int j = 0; j < nc[1]; ++j) {
      const int32_t* row = cv.grid + ((uint32_t)(c0[0] + i) * cv.syz +
                                      (uint32_t)(c0[1] + j) * cv.dz + (uint32_t)c0[2]);
      const int32_t v0 = __ldg(row);
      const int32_t v1 = nc[2] > 1 ? __ldg(row + 1) : -1;
      const int32_t v2 = nc[2] > 2 ? __ldg(row + 2) : -1;
      // all empty <=> each is -1 <=> their AND is -1 (an index >= 0 clears the sign bit)
      if ((v0 & v1 & v2) != -1) return false;
    }
  return true;
#else
  // up to 3 x 3 x 3 cells, every load issued at once (predicated): ONE memory
  // round trip instead of one per row (the row-by-row early exit took up to 9
  // dependent round trips per chunk; ncu: the culling pass was ~9 % of the
  // linearize kernel's stall samples for 4 % of its instructions).  All empty
  // <=> every value is -1 <=> their AND is -1 (an index >= 0 clears the sign bit)
  const int32_t* base = cv.grid + ((uint32_t)c0[0] * cv.syz + (uint32_t)c0[1] * cv.dz + (uint32_t)c0[2]);
  int32_t all = -1;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (i < nc[0] && j < nc[1] && k < nc[2])
          all &= __ldg(base + ((uint32_t)i * cv.syz + (uint32_t)j * cv.dz + (uint32_t)k));
  return all == -1;
#endif
}

// Culling bits for 32 chunks at once (whole warp, all lanes): lane j tests
// chunk c0 + j * stride of the cloud (chunks at or past `nchunks` count as
// culled: they hold no points).  Bit j of the result = chunk culled.
// cv: the map's coarsest level if its index is a dense grid, else nullptr (then
// only the map box test applies).
__device__ inline uint32_t cull_ballot(const float* __restrict__ chunk_box, int64_t c0, int stride,
                                       int64_t nchunks, const float* Rf, const double* t,
                                       const float* map_lo, const float* map_hi,
                                       const MapLevelDev* cv) {
  const int64_t c = c0 + (int64_t)(threadIdx.x & 31) * stride;
  bool cul = true;
  if (c < nchunks) {
    float box[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) box[j] = __ldg(chunk_box + 6 * c + j);
    cul = cv ? chunk_culled_grid(box, Rf, t, *cv) : chunk_culled(box, Rf, t, map_lo, map_hi);
  }
  return __ballot_sync(0xffffffffu, cul);
}

__device__ inline double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ inline int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// upper_bound(tile_start[0..num_factors], tile) - 1: the factor owning `tile`
// (factors with zero tiles are skipped).
__device__ inline int64_t owner_of_tile(const int32_t* tile_start, int64_t num_factors,
                                        int64_t tile) {
  int64_t lo = 0, hi = num_factors;  // tile_start[lo] <= tile < tile_start[hi]
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(tile_start + mid) <= tile) lo = mid; else hi = mid;
  }
  return lo;
}

}  // namespace gvox

// ---------------------------------------------------------------------------
// Packed fp32 pairs (sm_100a FFMA2 / FADD2 / FMUL2 via PTX f32x2).  A pair is
// held in one 64-bit register; ptxas folds scalar broadcasts (.F32), half
// swaps (.LO_HI) and negations into the packed instruction's operands.
// Round-to-nearest, no contraction beyond the explicit fma.
// ---------------------------------------------------------------------------
namespace gvox {
typedef unsigned long long f2_t;

__device__ __forceinline__ f2_t pk(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ f2_t bc(float a) { return pk(a, a); }
__device__ __forceinline__ float lo(f2_t v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a;
}
__device__ __forceinline__ float hi(f2_t v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return b;
}
__device__ __forceinline__ f2_t swp(f2_t v) { return pk(hi(v), lo(v)); }
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
  f2_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
}  // namespace gvox
