// k_knn.cu -- GPU preprocessing: exact k nearest
// neighbours ("the costly exact nearest neighbor search is only
// performed in the preprocessing step") and the per-point covariance from
// them, GICP plane-regularized (readings R26-R28).
//
// B200 design: points of each cloud are counting-sorted into a uniform cell
// grid (count -> exclusive scan -> scatter of 16 B {x, y, z, index} records),
// so a cell's points are one contiguous run.  Queries walk the SORTED order
// (a warp's 32 queries are spatial neighbours, so they read the same cells),
// each thread searching rings of cells (Chebyshev distance R = 0, 1, 2, ...)
// with its top-k list in registers, and stopping once the k-th distance is
// certainly below the distance to every unsearched cell.  Distances are fp64
// with a pinned, unfused operation order (R26), so the k-set and its order
// are exactly the oracle's.
#include <cstdint>
#include <cstdlib>

#include "k_common.cuh"

namespace gvox {
namespace {

constexpr int kKnnThreads = 64;

__device__ __forceinline__ double sq_dist_pinned(float px, float py, float pz, float qx, float qy,
                                                 float qz) {
  const double dx = __dsub_rn((double)qx, (double)px);
  const double dy = __dsub_rn((double)qy, (double)py);
  const double dz = __dsub_rn((double)qz, (double)pz);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// fp32 pre-filter of the insertion test (exact): the fp32 squared distance
// (three rounded differences, squares and sums: relative error below 6 * 2^-24
// for finite inputs without underflow) exceeds the fp64 gate by more than that
// error only if the pinned fp64 distance (relative error ~2^-51) does too, so
// a candidate rejected here would have been rejected by `d2 < gate` -- the
// fp64 distance is computed only for the candidates that might enter the list.
// gate32(g) = an upper bound of g * (1 + 2^-20) in fp32 (+inf stays +inf; the
// absolute 1e-30 covers underflowing squares).
__device__ __forceinline__ float gate32(double g) {
  return __double2float_ru(fma(g, 9.5367431640625e-07, g)) + 1e-30f;
}
__device__ __forceinline__ float sq_dist_f32(float px, float py, float pz, float qx, float qy,
                                             float qz) {
  const float dx = qx - px, dy = qy - py, dz = qz - pz;
  return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
}

// (j == km1) ? a : b through PTX selp: opaque to the compiler, so an unrolled
// `for j: if (j == k - 1) x = list[j]` is not folded back into the dynamic
// index list[k - 1], which would move the whole top-k list into local memory
__device__ __forceinline__ double sel_eq(int j, int km1, double a, double b) {
  double r;
  asm("{ .reg .pred p; setp.eq.s32 p, %1, %2; selp.f64 %0, %3, %4, p; }"
      : "=d"(r) : "r"(j), "r"(km1), "d"(a), "d"(b));
  return r;
}
__device__ __forceinline__ int32_t sel_eq(int j, int km1, int32_t a, int32_t b) {
  int32_t r;
  asm("{ .reg .pred p; setp.eq.s32 p, %1, %2; selp.b32 %0, %3, %4, p; }"
      : "=r"(r) : "r"(j), "r"(km1), "r"(a), "r"(b));
  return r;
}

__device__ __forceinline__ int32_t cell_coord(float x, double lo, double inv_s, int32_t dim) {
  int32_t c = __double2int_rd(((double)x - lo) * inv_s);
  return min(max(c, 0), dim - 1);
}

// per point: cloud-grid cell (global cell index) and its count
__global__ void k_knn_count(const float* __restrict__ pts, const KnnCloudDev* __restrict__ clouds,
                            const int32_t* __restrict__ tile_start, const int32_t* __restrict__ tile_cloud,
                            int tile_pts, int32_t* __restrict__ cell_of, int32_t* __restrict__ count) {
  const int32_t c = __ldg(tile_cloud + blockIdx.x);
  const KnnCloudDev cd = clouds[c];
  const int64_t k = cd.first + (int64_t)(blockIdx.x - __ldg(tile_start + c)) * tile_pts + threadIdx.x;
  for (int64_t i = k; i < cd.first + cd.n && i < k - threadIdx.x + tile_pts; i += blockDim.x) {
    const float x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    const int32_t cx = cell_coord(x, cd.lo[0], cd.inv_s, cd.dim[0]);
    const int32_t cy = cell_coord(y, cd.lo[1], cd.inv_s, cd.dim[1]);
    const int32_t cz = cell_coord(z, cd.lo[2], cd.inv_s, cd.dim[2]);
    const int32_t cell = cd.cell0 + (cx * cd.dim[1] + cy) * cd.dim[2] + cz;
    cell_of[i] = cell;
    atomicAdd(count + cell, 1);
  }
}

// scatter into cell order: {x, y, z, local index bits}
__global__ void k_knn_scatter(const float* __restrict__ pts, const KnnCloudDev* __restrict__ clouds,
                              const int32_t* __restrict__ tile_start, const int32_t* __restrict__ tile_cloud,
                              int tile_pts, const int32_t* __restrict__ cell_of,
                              const int32_t* __restrict__ cell_start, int32_t* __restrict__ fill,
                              float4* __restrict__ sorted) {
  const int32_t c = __ldg(tile_cloud + blockIdx.x);
  const KnnCloudDev cd = clouds[c];
  const int64_t k = cd.first + (int64_t)(blockIdx.x - __ldg(tile_start + c)) * tile_pts + threadIdx.x;
  for (int64_t i = k; i < cd.first + cd.n && i < k - threadIdx.x + tile_pts; i += blockDim.x) {
    const int32_t cell = cell_of[i];
    const int32_t slot = cell_start[cell] + atomicAdd(fill + cell, 1);
    sorted[slot] = make_float4(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2],
                               __int_as_float((int32_t)(i - cd.first)));
  }
}

// per-cloud bounding box (order-preserving int encoding; box[6 c ..] =
// min xyz, max xyz, initialised to INT_MAX / INT_MIN); non-finite -> flag
__global__ void k_knn_bbox(const float* __restrict__ pts, const KnnCloudDev* __restrict__ clouds,
                           const int32_t* __restrict__ tile_start, const int32_t* __restrict__ tile_cloud,
                           int tile_pts, int32_t* __restrict__ box, int32_t* __restrict__ bad) {
  const int32_t c = __ldg(tile_cloud + blockIdx.x);
  const KnnCloudDev cd = clouds[c];
  const int64_t k = cd.first + (int64_t)(blockIdx.x - __ldg(tile_start + c)) * tile_pts + threadIdx.x;
  int32_t mn[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, mx[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
  int nonfinite = 0;
  for (int64_t i = k; i < cd.first + cd.n && i < k - threadIdx.x + tile_pts; i += blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float x = pts[3 * i + a];
      nonfinite |= !isfinite(x);
      const int32_t o = float_to_ordered(x);
      mn[a] = min(mn[a], o);
      mx[a] = max(mx[a], o);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
  }
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (mn[a] != INT32_MAX) atomicMin(box + 6 * c + a, mn[a]);
      if (mx[a] != INT32_MIN) atomicMax(box + 6 * c + 3 + a, mx[a]);
    }
    if (nonfinite) atomicOr(bad, 1);
  }
}

// Exact k-NN: one thread per query, queries in cell-sorted order.
template <int MAXK>
__global__ void __launch_bounds__(kKnnThreads)
    k_knn_query(const KnnCloudDev* __restrict__ clouds, const int32_t* __restrict__ tile_start,
                const int32_t* __restrict__ tile_cloud, int tile_pts, const float4* __restrict__ sorted,
                const int32_t* __restrict__ cell_start, int k, int32_t* __restrict__ out) {
  const int32_t c = __ldg(tile_cloud + blockIdx.x);
  const KnnCloudDev cd = clouds[c];
  const int64_t t0 = cd.first + (int64_t)(blockIdx.x - __ldg(tile_start + c)) * tile_pts;
  for (int64_t t = t0 + threadIdx.x; t < cd.first + cd.n && t < t0 + tile_pts; t += blockDim.x) {
    const float4 q = sorted[t];
    const int32_t qi = __float_as_int(q.w);
    const int32_t cx = cell_coord(q.x, cd.lo[0], cd.inv_s, cd.dim[0]);
    const int32_t cy = cell_coord(q.y, cd.lo[1], cd.inv_s, cd.dim[1]);
    const int32_t cz = cell_coord(q.z, cd.lo[2], cd.inv_s, cd.dim[2]);
    double bd[MAXK];
    int32_t bi[MAXK];
#pragma unroll
    for (int j = 0; j < MAXK; ++j) {
      bd[j] = __longlong_as_double(0x7ff0000000000000ll);  // +inf
      bi[j] = INT32_MAX;
    }
    int found = 0;
    double kth = __longlong_as_double(0x7ff0000000000000ll);  // (bd, bi)[k - 1]: the insertion gate
    int32_t kidx = INT32_MAX;
    float kth32 = __int_as_float(0x7f800000);  // gate32(kth)
    // slack for the cell assignment's rounding (floor((x - lo) / s) in fp64)
    const double slack = 1e-9 * (fabs(cd.lo[0]) + fabs(cd.lo[1]) + fabs(cd.lo[2]) +
                                 cd.s * (cd.dim[0] + cd.dim[1] + cd.dim[2]) + 1.0);
    const double s = cd.s;
    for (int R = 0;; ++R) {
      const int32_t x0 = max(cx - R, 0), x1 = min(cx + R, cd.dim[0] - 1);
      const int32_t y0 = max(cy - R, 0), y1 = min(cy + R, cd.dim[1] - 1);
      const int32_t z0 = max(cz - R, 0), z1 = min(cz + R, cd.dim[2] - 1);
      // the cells of one (x, y) column are consecutive in the grid and so are
      // their points in `sorted`: a column's new cells are one or two runs
      auto scan_run = [&](int32_t c0, int32_t c1) {  // cells [c0, c1] of one column
        const int32_t s0 = __ldg(cell_start + c0), s1 = __ldg(cell_start + c1 + 1);
        for (int32_t si = s0; si < s1; ++si) {
          const float4 p = __ldg(sorted + si);
          ++found;
          if (sq_dist_f32(p.x, p.y, p.z, q.x, q.y, q.z) > kth32) continue;
          const double d2 = sq_dist_pinned(q.x, q.y, q.z, p.x, p.y, p.z);
          const int32_t pi = __float_as_int(p.w);
          if (d2 < kth || (d2 == kth && pi < kidx)) {
            // insertion into the (d2, index)-sorted list (registers: unrolled)
            double cd2 = d2;
            int32_t ci = pi;
#pragma unroll
            for (int j = 0; j < MAXK; ++j) {
              const bool lt = cd2 < bd[j] || (cd2 == bd[j] && ci < bi[j]);
              const double td = bd[j];
              const int32_t ti = bi[j];
              bd[j] = lt ? cd2 : td;
              bi[j] = lt ? ci : ti;
              cd2 = lt ? td : cd2;
              ci = lt ? ti : ci;
            }
#pragma unroll
            for (int j = 0; j < MAXK; ++j) {
              kth = sel_eq(j, k - 1, bd[j], kth);
              kidx = sel_eq(j, k - 1, bi[j], kidx);
            }
            kth32 = gate32(kth);
          }
        }
      };
      for (int32_t x = x0; x <= x1; ++x) {
        const double bx0 = cd.lo[0] + (double)x * s;
        const double ex = fmax(fmax(bx0 - (double)q.x, (double)q.x - (bx0 + s)), 0.0);
        for (int32_t y = y0; y <= y1; ++y) {
          const bool face = (x == cx - R) | (x == cx + R) | (y == cy - R) | (y == cy + R);
          if (found >= k) {  // exact pruning of the whole column by its xy distance
            const double by0 = cd.lo[1] + (double)y * s;
            const double ey = fmax(fmax(by0 - (double)q.y, (double)q.y - (by0 + s)), 0.0);
            const double em = fmax(sqrt(ex * ex + ey * ey) - slack, 0.0);
            if (em * em > kth * (1.0 + 1e-9)) continue;
          }
          const int32_t col = cd.cell0 + (x * cd.dim[1] + y) * cd.dim[2];
          if (face) {
            scan_run(col + z0, col + z1);
          } else {  // interior column: only z = cz - R and cz + R are new
            if (cz - R >= z0) scan_run(col + cz - R, col + cz - R);
            if (cz + R <= z1) scan_run(col + cz + R, col + cz + R);
          }
        }
      }
      // every unsearched point lies beyond the searched cube's faces that are
      // inside the grid; stop once the k-th distance is certainly below that
      const bool all = x0 == 0 && y0 == 0 && z0 == 0 && x1 == cd.dim[0] - 1 &&
                       y1 == cd.dim[1] - 1 && z1 == cd.dim[2] - 1;
      if (all) break;
      if (found >= k) {
        double b = __longlong_as_double(0x7ff0000000000000ll);
        const int32_t cc[3] = {cx, cy, cz};
        const float qq[3] = {q.x, q.y, q.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (cc[a] - R > 0) b = fmin(b, (double)qq[a] - (cd.lo[a] + (double)(cc[a] - R) * s));
          if (cc[a] + R < cd.dim[a] - 1) b = fmin(b, cd.lo[a] + (double)(cc[a] + R + 1) * s - (double)qq[a]);
        }
        b -= slack;
        if (b > 0.0 && kth < b * b * (1.0 - 1e-9)) break;
      }
    }
    int32_t* row = out + (cd.first + qi) * (int64_t)k;
#pragma unroll
    for (int j = 0; j < MAXK; ++j)
      if (j < k) row[j] = bi[j] == INT32_MAX ? -1 : bi[j];
  }
}

// Exact k-NN with G lanes per query (k <= MAXK): the same ring search and
// pinned distances as k_knn_query, but each ring's candidate points are split
// over the query's G lanes (lane g takes points g, g + G, ... of every cell
// run), each lane keeping its own sorted (d2, index) list.  At the end of a
// ring the group merges the lists -- k rounds of a group-wide minimum over the
// lanes' heads, the winner popping its head -- into lane 0 (the other lanes
// restart empty, so no point is counted twice), and every lane keeps the merged
// k-th entry, the bound the next ring prunes and stops with.  A point set and
// its order are unique under (d2, index), so the result is exactly
// k_knn_query's (and the oracle's); only the in-ring column pruning uses the
// previous ring's bound.  G x more threads per frame: the search of one
// odometry frame no longer leaves the GPU nearly empty.
template <int MAXK, int G>
__global__ void __launch_bounds__(kKnnThreads)
    k_knn_query_g(const KnnCloudDev* __restrict__ clouds, const int32_t* __restrict__ tile_start,
                  const int32_t* __restrict__ tile_cloud, int tile_pts, const float4* __restrict__ sorted,
                  const int32_t* __restrict__ cell_start, int k, int32_t* __restrict__ out) {
  static_assert(G == 2 || G == 4 || G == 8 || G == 16 || G == 32, "G: a power of two <= 32");
  // G CTAs per tile of the plan (one query per thread of a 64-thread CTA):
  // CTA part p of tile T takes the tile's queries [p, p + 1) * tile_pts / G
  const int64_t tile = blockIdx.x / G;
  const int part = (int)(blockIdx.x % G);
  const int32_t c = __ldg(tile_cloud + tile);
  const KnnCloudDev cd = clouds[c];
  const int per = tile_pts / G;
  const int64_t t0 = cd.first + (int64_t)(tile - __ldg(tile_start + c)) * tile_pts + (int64_t)part * per;
  const int lane = threadIdx.x & 31, sub = lane & (G - 1);
  const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (lane & ~(G - 1));
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const int64_t tend = min(cd.first + cd.n, t0 + (int64_t)per);
  // (the G lanes of a query run the same iterations: the group stays converged
  // at every merge)
  for (int64_t t = t0 + threadIdx.x / G; t < tend; t += blockDim.x / G) {
    const float4 q = sorted[t];
    const int32_t qi = __float_as_int(q.w);
    const int32_t cx = cell_coord(q.x, cd.lo[0], cd.inv_s, cd.dim[0]);
    const int32_t cy = cell_coord(q.y, cd.lo[1], cd.inv_s, cd.dim[1]);
    const int32_t cz = cell_coord(q.z, cd.lo[2], cd.inv_s, cd.dim[2]);
    double bd[MAXK];
    int32_t bi[MAXK];
#pragma unroll
    for (int j = 0; j < MAXK; ++j) {
      bd[j] = kInf;
      bi[j] = INT32_MAX;
    }
    int found_g = 0;    // candidates the group has scanned before this ring
    double kth = kInf;  // the merged list's k-th (d2, index)
    int32_t kidx = INT32_MAX;
    const double slack = 1e-9 * (fabs(cd.lo[0]) + fabs(cd.lo[1]) + fabs(cd.lo[2]) +
                                 cd.s * (cd.dim[0] + cd.dim[1] + cd.dim[2]) + 1.0);
    const double s = cd.s;
    for (int R = 0;; ++R) {
      const int32_t x0 = max(cx - R, 0), x1 = min(cx + R, cd.dim[0] - 1);
      const int32_t y0 = max(cy - R, 0), y1 = min(cy + R, cd.dim[1] - 1);
      const int32_t z0 = max(cz - R, 0), z1 = min(cz + R, cd.dim[2] - 1);
      int found = 0;
      // the gate: the smaller of this lane's own k-th and the merged bound
      double gth = kth;
      int32_t gidx = kidx;
      float gth32 = gate32(gth);
      auto scan_run = [&](int32_t c0, int32_t c1) {
        const int32_t s0 = __ldg(cell_start + c0), s1 = __ldg(cell_start + c1 + 1);
        for (int32_t si = s0 + sub; si < s1; si += G) {
          const float4 p = __ldg(sorted + si);
          ++found;
          if (sq_dist_f32(p.x, p.y, p.z, q.x, q.y, q.z) > gth32) continue;
          const double d2 = sq_dist_pinned(q.x, q.y, q.z, p.x, p.y, p.z);
          const int32_t pi = __float_as_int(p.w);
          if (d2 < gth || (d2 == gth && pi < gidx)) {
            double cd2 = d2;
            int32_t ci = pi;
#pragma unroll
            for (int j = 0; j < MAXK; ++j) {
              const bool lt = cd2 < bd[j] || (cd2 == bd[j] && ci < bi[j]);
              const double td = bd[j];
              const int32_t ti = bi[j];
              bd[j] = lt ? cd2 : td;
              bi[j] = lt ? ci : ti;
              cd2 = lt ? td : cd2;
              ci = lt ? ti : ci;
            }
            // the own list's k-th, if it is below the merged bound
            double ok = kInf;
            int32_t oi = INT32_MAX;
#pragma unroll
            for (int j = 0; j < MAXK; ++j) {
              ok = sel_eq(j, k - 1, bd[j], ok);
              oi = sel_eq(j, k - 1, bi[j], oi);
            }
            if (ok < gth || (ok == gth && oi < gidx)) {
              gth = ok;
              gidx = oi;
            }
            gth32 = gate32(gth);
          }
        }
      };
      for (int32_t x = x0; x <= x1; ++x) {
        const double bx0 = cd.lo[0] + (double)x * s;
        const double ex = fmax(fmax(bx0 - (double)q.x, (double)q.x - (bx0 + s)), 0.0);
        for (int32_t y = y0; y <= y1; ++y) {
          const bool face = (x == cx - R) | (x == cx + R) | (y == cy - R) | (y == cy + R);
          if (found_g >= k) {  // exact pruning of the whole column by the merged bound
            const double by0 = cd.lo[1] + (double)y * s;
            const double ey = fmax(fmax(by0 - (double)q.y, (double)q.y - (by0 + s)), 0.0);
            const double em = fmax(sqrt(ex * ex + ey * ey) - slack, 0.0);
            if (em * em > kth * (1.0 + 1e-9)) continue;
          }
          const int32_t col = cd.cell0 + (x * cd.dim[1] + y) * cd.dim[2];
          if (face) {
            scan_run(col + z0, col + z1);
          } else {
            if (cz - R >= z0) scan_run(col + cz - R, col + cz - R);
            if (cz + R <= z1) scan_run(col + cz + R, col + cz + R);
          }
        }
      }
      // ---- merge: round j takes the group minimum of the lanes' heads (all
      // MAXK rounds, every index static: the lists stay in registers; rounds
      // past k merge entries nobody reads)
      __syncwarp(gmask);
      double md[MAXK];
      int32_t mi[MAXK];
#pragma unroll
      for (int j = 0; j < MAXK; ++j) {
        double hd = bd[0];
        int32_t hi = bi[0];
        int who = sub;
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
          const double od = __shfl_xor_sync(gmask, hd, o, G);
          const int32_t oi = __shfl_xor_sync(gmask, hi, o, G);
          const int ow = __shfl_xor_sync(gmask, who, o, G);
          if (od < hd || (od == hd && oi < hi)) {
            hd = od;
            hi = oi;
            who = ow;
          }
        }
        const bool pop = who == sub;  // the winner pops its head
#pragma unroll
        for (int m = 0; m < MAXK - 1; ++m) {
          bd[m] = pop ? bd[m + 1] : bd[m];
          bi[m] = pop ? bi[m + 1] : bi[m];
        }
        bd[MAXK - 1] = pop ? kInf : bd[MAXK - 1];
        bi[MAXK - 1] = pop ? INT32_MAX : bi[MAXK - 1];
        md[j] = hd;
        mi[j] = hi;
      }
#pragma unroll
      for (int j = 0; j < MAXK; ++j) {
        kth = sel_eq(j, k - 1, md[j], kth);
        kidx = sel_eq(j, k - 1, mi[j], kidx);
      }
      // lane 0 holds the merged list, the others start the next ring empty
#pragma unroll
      for (int j = 0; j < MAXK; ++j) {
        bd[j] = sub == 0 ? md[j] : kInf;
        bi[j] = sub == 0 ? mi[j] : INT32_MAX;
      }
      found_g += __reduce_add_sync(gmask, found);
      // every unsearched point lies beyond the searched cube's faces that are
      // inside the grid; stop once the k-th distance is certainly below that
      const bool all = x0 == 0 && y0 == 0 && z0 == 0 && x1 == cd.dim[0] - 1 &&
                       y1 == cd.dim[1] - 1 && z1 == cd.dim[2] - 1;
      if (all) break;
      if (found_g >= k) {
        double b = kInf;
        const int32_t cc[3] = {cx, cy, cz};
        const float qq[3] = {q.x, q.y, q.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (cc[a] - R > 0) b = fmin(b, (double)qq[a] - (cd.lo[a] + (double)(cc[a] - R) * s));
          if (cc[a] + R < cd.dim[a] - 1) b = fmin(b, cd.lo[a] + (double)(cc[a] + R + 1) * s - (double)qq[a]);
        }
        b -= slack;
        if (b > 0.0 && kth < b * b * (1.0 - 1e-9)) break;
      }
    }
    if (sub == 0) {
      int32_t* row = out + (cd.first + qi) * (int64_t)k;
#pragma unroll
      for (int j = 0; j < MAXK; ++j)
        if (j < k) row[j] = bi[j] == INT32_MAX ? -1 : bi[j];
    }
  }
}

// symmetric 3x3 (a00 a01 a02 a11 a12 a22) -> unit eigenvector of the smallest
// eigenvalue, cyclic Jacobi in fp64 (converges to rounding level)
__device__ void smallest_eigvec(const double* A6, double* v) {
  double a[3][3] = {{A6[0], A6[1], A6[2]}, {A6[1], A6[3], A6[4]}, {A6[2], A6[4], A6[5]}};
  double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 12; ++sweep) {
    const double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    const double dia = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]);
    if (off <= 1e-300 || off <= 1e-18 * dia) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, r = pq == 0 ? 1 : 2;
      if (a[p][r] == 0.0) continue;
      const double theta = (a[r][r] - a[p][p]) / (2.0 * a[p][r]);
      const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
      for (int j = 0; j < 3; ++j) {  // A <- A J (columns p, r)
        const double ajp = a[j][p], ajr = a[j][r];
        a[j][p] = cs * ajp - sn * ajr;
        a[j][r] = sn * ajp + cs * ajr;
      }
      for (int j = 0; j < 3; ++j) {  // A <- J^T A (rows p, r)
        const double apj = a[p][j], arj = a[r][j];
        a[p][j] = cs * apj - sn * arj;
        a[r][j] = sn * apj + cs * arj;
      }
      for (int j = 0; j < 3; ++j) {
        const double vjp = V[j][p], vjr = V[j][r];
        V[j][p] = cs * vjp - sn * vjr;
        V[j][r] = sn * vjp + cs * vjr;
      }
    }
  }
  int m = 0;
  if (a[1][1] < a[m][m]) m = 1;
  if (a[2][2] < a[m][m]) m = 2;
  const double nv = sqrt(V[0][m] * V[0][m] + V[1][m] * V[1][m] + V[2][m] * V[2][m]);
  for (int j = 0; j < 3; ++j) v[j] = V[j][m] / nv;
}

// per point: sample covariance of its neighbours (fp64), smallest eigenvector
// oriented toward the cloud origin, C = I - (1 - 1e-3) n n^T (R27/R28)
__global__ void k_covariance(const float* __restrict__ pts, const KnnCloudDev* __restrict__ clouds,
                             const int32_t* __restrict__ tile_start, const int32_t* __restrict__ tile_cloud,
                             int tile_pts, const int32_t* __restrict__ nbr, int k,
                             float* __restrict__ cov, float* __restrict__ nrm) {
  const int32_t c = __ldg(tile_cloud + blockIdx.x);
  const KnnCloudDev cd = clouds[c];
  const int64_t k0 = cd.first + (int64_t)(blockIdx.x - __ldg(tile_start + c)) * tile_pts + threadIdx.x;
  for (int64_t i = k0; i < cd.first + cd.n && i < k0 - threadIdx.x + tile_pts; i += blockDim.x) {
    const int32_t* row = nbr + i * (int64_t)k;
    double m[3] = {0, 0, 0};
    int cnt = 0;
    for (int j = 0; j < k; ++j) {
      const int32_t q = row[j];
      if (q < 0) continue;
      const float* p = pts + 3 * (cd.first + q);
      m[0] += p[0];
      m[1] += p[1];
      m[2] += p[2];
      ++cnt;
    }
    double S[6] = {0, 0, 0, 0, 0, 0};
    if (cnt > 0) {
      for (int a = 0; a < 3; ++a) m[a] /= cnt;
      for (int j = 0; j < k; ++j) {
        const int32_t q = row[j];
        if (q < 0) continue;
        const float* p = pts + 3 * (cd.first + q);
        const double dx = p[0] - m[0], dy = p[1] - m[1], dz = p[2] - m[2];
        S[0] += dx * dx;
        S[1] += dx * dy;
        S[2] += dx * dz;
        S[3] += dy * dy;
        S[4] += dy * dz;
        S[5] += dz * dz;
      }
      for (int a = 0; a < 6; ++a) S[a] /= cnt;
    }
    float* co = cov + 6 * i;
    float* no = nrm + 3 * i;
    if (S[0] == 0.0 && S[1] == 0.0 && S[2] == 0.0 && S[3] == 0.0 && S[4] == 0.0 && S[5] == 0.0) {
      co[0] = 1e-6f; co[1] = 0.f; co[2] = 0.f; co[3] = 1e-6f; co[4] = 0.f; co[5] = 1e-6f;
      no[0] = no[1] = no[2] = 0.f;
      continue;
    }
    double v[3];
    smallest_eigvec(S, v);
    const float* pi = pts + 3 * i;
    if (v[0] * pi[0] + v[1] * pi[1] + v[2] * pi[2] > 0.0) {
      v[0] = -v[0];
      v[1] = -v[1];
      v[2] = -v[2];
    }
    const double e = 1.0 - 1e-3;
    co[0] = (float)(1.0 - e * v[0] * v[0]);
    co[1] = (float)(-e * v[0] * v[1]);
    co[2] = (float)(-e * v[0] * v[2]);
    co[3] = (float)(1.0 - e * v[1] * v[1]);
    co[4] = (float)(-e * v[1] * v[2]);
    co[5] = (float)(1.0 - e * v[2] * v[2]);
    no[0] = (float)v[0];
    no[1] = (float)v[1];
    no[2] = (float)v[2];
  }
}

// ---- exclusive scan of int32 counts (3 phases; any length < 2^31)
constexpr int kScanThreads = 1024, kScanPer = 4, kScanBlock = kScanThreads * kScanPer;

__device__ __forceinline__ int32_t block_exclusive_scan(int32_t v, int32_t* warp_s, int32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_s[w] = x;
  __syncthreads();
  if (w == 0) {
    int32_t s = lane < (int)(blockDim.x >> 5) ? warp_s[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_s[lane] = s;  // inclusive warp prefix
  }
  __syncthreads();
  const int32_t before = w > 0 ? warp_s[w - 1] : 0;
  if (total) *total = warp_s[(blockDim.x >> 5) - 1];
  return before + x - v;
}

__global__ void __launch_bounds__(kScanThreads)
    k_scan_blocks(const int32_t* __restrict__ in, int64_t n, int32_t* __restrict__ out,
                  int32_t* __restrict__ sums) {
  __shared__ int32_t warp_s[32];
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + (int64_t)threadIdx.x * kScanPer;
  int32_t v[kScanPer], t = 0;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    v[j] = base + j < n ? in[base + j] : 0;
    t += v[j];
  }
  int32_t total;
  int32_t ex = block_exclusive_scan(t, warp_s, &total);
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    if (base + j < n) out[base + j] = ex;
    ex += v[j];
  }
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// one block: exclusive scan of the block sums in chunks (carry across chunks);
// also writes the grand total to out_total
__global__ void __launch_bounds__(kScanThreads)
    k_scan_sums(int32_t* __restrict__ sums, int64_t nb, int32_t* __restrict__ out_total) {
  __shared__ int32_t warp_s[32];
  __shared__ int32_t carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nb; b0 += kScanThreads) {
    const int64_t i = b0 + threadIdx.x;
    const int32_t v = i < nb ? sums[i] : 0;
    int32_t total;
    const int32_t ex = block_exclusive_scan(v, warp_s, &total);
    const int32_t carry = carry_s;
    if (i < nb) sums[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *out_total = carry_s;
}

__global__ void k_scan_add(int32_t* __restrict__ out, int64_t n, const int32_t* __restrict__ sums) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += sums[i / kScanBlock];
}

}  // namespace

// out[0..n) = exclusive prefix sums of in, out[n] = total.  scratch: ceil(n / 4096) ints.
void launch_exclusive_scan(const int32_t* in, int64_t n, int32_t* out, int32_t* scratch,
                           cudaStream_t stream) {
  const int64_t nb = (n + kScanBlock - 1) / kScanBlock;
  if (nb > 0) {
    k_scan_blocks<<<(unsigned)nb, kScanThreads, 0, stream>>>(in, n, out, scratch);
    note_launch();
  }
  k_scan_sums<<<1, kScanThreads, 0, stream>>>(scratch, nb, out + n);
  note_launch();
  if (nb > 1) {
    k_scan_add<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(out, n, scratch);
    note_launch();
  }
}

void launch_knn_bbox(const float* pts, const KnnCloudDev* clouds, const int32_t* tile_start,
                     const int32_t* tile_cloud, int64_t num_tiles, int tile_pts, int32_t* box,
                     int32_t* bad, cudaStream_t stream) {
  if (num_tiles <= 0) return;
  k_knn_bbox<<<(unsigned)num_tiles, 256, 0, stream>>>(pts, clouds, tile_start, tile_cloud, tile_pts,
                                                     box, bad);
  note_launch();
}

void launch_knn_count(const float* pts, const KnnCloudDev* clouds, const int32_t* tile_start,
                      const int32_t* tile_cloud, int64_t num_tiles, int tile_pts, int32_t* cell_of,
                      int32_t* count, cudaStream_t stream) {
  if (num_tiles <= 0) return;
  k_knn_count<<<(unsigned)num_tiles, 256, 0, stream>>>(pts, clouds, tile_start, tile_cloud, tile_pts,
                                                      cell_of, count);
  note_launch();
}

void launch_knn_scatter(const float* pts, const KnnCloudDev* clouds, const int32_t* tile_start,
                        const int32_t* tile_cloud, int64_t num_tiles, int tile_pts,
                        const int32_t* cell_of, const int32_t* cell_start, int32_t* fill,
                        float4* sorted, cudaStream_t stream) {
  if (num_tiles <= 0) return;
  k_knn_scatter<<<(unsigned)num_tiles, 256, 0, stream>>>(pts, clouds, tile_start, tile_cloud, tile_pts,
                                                        cell_of, cell_start, fill, sorted);
  note_launch();
}

void launch_knn_query(const KnnCloudDev* clouds, const int32_t* tile_start, const int32_t* tile_cloud,
                      int64_t num_tiles, int tile_pts, const float4* sorted,
                      const int32_t* cell_start, int k, int32_t* out, cudaStream_t stream) {
  if (num_tiles <= 0) return;
  // lanes per query: a batch of at most ~64k queries (one or a few odometry
  // frames) leaves the GPU mostly idle at one thread per query, so it uses 4
  // (r02m, one 15.6k-point frame: 193 -> 142 us, issue-active 20 -> 34 %);
  // larger batches fill the GPU already and keep 1 (C3's 0.8 M points: 2.31 ms
  // at G = 1, 4.21 at G = 4).  GVOX_KNN_GROUP overrides (1, 4, 8).
  // (r02aq, one 15.6k-point frame: G = 8 0.112 ms vs G = 4 0.117 ms; r02bj:
  // G = 16 0.120 ms -- the merges cost more than the extra lanes give)
  const int64_t nq = (int64_t)num_tiles * tile_pts;
  int kGroup = nq <= (32 << 10) ? 8 : nq <= (64 << 10) ? 4 : 1;
  if (const char* e = std::getenv("GVOX_KNN_GROUP")) kGroup = std::atoi(e);
  if (k <= 10 && kGroup == 16 && tile_pts % 16 == 0)
    k_knn_query_g<10, 16><<<(unsigned)(num_tiles * 16), kKnnThreads, 0, stream>>>(
        clouds, tile_start, tile_cloud, tile_pts, sorted, cell_start, k, out);
  else if (k <= 10 && kGroup == 8 && tile_pts % 8 == 0)
    k_knn_query_g<10, 8><<<(unsigned)(num_tiles * 8), kKnnThreads, 0, stream>>>(
        clouds, tile_start, tile_cloud, tile_pts, sorted, cell_start, k, out);
  else if (k <= 10 && kGroup == 4 && tile_pts % 4 == 0)
    k_knn_query_g<10, 4><<<(unsigned)(num_tiles * 4), kKnnThreads, 0, stream>>>(
        clouds, tile_start, tile_cloud, tile_pts, sorted, cell_start, k, out);
  else if (k <= 10)
    k_knn_query<10><<<(unsigned)num_tiles, kKnnThreads, 0, stream>>>(clouds, tile_start, tile_cloud,
                                                                     tile_pts, sorted, cell_start, k, out);
  else if (k <= 16 && kGroup == 8 && tile_pts % 8 == 0)
    k_knn_query_g<16, 8><<<(unsigned)(num_tiles * 8), kKnnThreads, 0, stream>>>(
        clouds, tile_start, tile_cloud, tile_pts, sorted, cell_start, k, out);
  else if (k <= 16 && kGroup == 4 && tile_pts % 4 == 0)
    k_knn_query_g<16, 4><<<(unsigned)(num_tiles * 4), kKnnThreads, 0, stream>>>(
        clouds, tile_start, tile_cloud, tile_pts, sorted, cell_start, k, out);
  else if (k <= 16)
    k_knn_query<16><<<(unsigned)num_tiles, kKnnThreads, 0, stream>>>(clouds, tile_start, tile_cloud,
                                                                     tile_pts, sorted, cell_start, k, out);
  else
    k_knn_query<32><<<(unsigned)num_tiles, kKnnThreads, 0, stream>>>(clouds, tile_start, tile_cloud,
                                                                     tile_pts, sorted, cell_start, k, out);
  note_launch();
}

void launch_covariance(const float* pts, const KnnCloudDev* clouds, const int32_t* tile_start,
                       const int32_t* tile_cloud, int64_t num_tiles, int tile_pts, const int32_t* nbr,
                       int k, float* cov, float* nrm, cudaStream_t stream) {
  if (num_tiles <= 0) return;
  k_covariance<<<(unsigned)num_tiles, 64, 0, stream>>>(pts, clouds, tile_start, tile_cloud, tile_pts,
                                                       nbr, k, cov, nrm);
  note_launch();
}

}  // namespace gvox
