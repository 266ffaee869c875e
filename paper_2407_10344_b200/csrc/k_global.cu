// k_global.cu -- global Gauss-Newton system of a factor graph of matching cost
// factors and its GPU solve (global mapping P:391, the
// CPU solver's share of the optimisation P:814).
//
//   H = sum_f scatter(H_f),  b = sum_f scatter(b_f)  over the VARIABLE poses,
//   (H + lambda I) delta = -b  by block-Jacobi preconditioned conjugate
//   gradients in fp64.
//
// Layout: block-sparse rows (BSR, 6x6 fp64 blocks, both (i, j) and (j, i)
// stored, columns ascending per row).  Every block and every right-hand-side
// entry is summed by one warp / thread over its contribution list in
// ascending factor order: the system is bitwise deterministic.  The PCG runs
// as ONE cooperative persistent kernel (k_pcg_persistent: grid barriers
// between SpMV, update and direction phases); the two-kernel version as the
// body of a CUDA graph WHILE node (k_spmv_dot -> k_pcg_update, the latter
// sets the condition) is kept behind GVOX_PCG_GRAPH=1 for comparison.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "k_common.cuh"

namespace cg = cooperative_groups;

namespace gvox {
namespace {

constexpr int kUpdThreads = 1024;

// one warp per block: sum its contributions (factor, kind) in order
__global__ void k_assemble_blocks(const gvox_linear_factor* __restrict__ rec,
                                  const int32_t* __restrict__ contrib_start,
                                  const int32_t* __restrict__ contrib, int64_t num_blocks,
                                  const uint8_t* __restrict__ is_diag, double lambda,
                                  double* __restrict__ blocks) {
  const int lane = threadIdx.x & 31;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= num_blocks) return;
  for (int e = lane; e < 36; e += 32) {
    double s = 0.0;
    for (int32_t c = contrib_start[b]; c < contrib_start[b + 1]; ++c) {
      const int32_t v = contrib[c];
      const int32_t f = v >> 2, kind = v & 3;
      const gvox_linear_factor& r = rec[f];
      const int rr = e / 6, cc = e % 6;
      s += kind == 0 ? r.H_ii[e] : kind == 1 ? r.H_ij[e] : kind == 2 ? r.H_ij[cc * 6 + rr] : r.H_jj[e];
    }
    if (is_diag[b] && (e % 7) == 0) s += lambda;
    blocks[36 * b + e] = s;
  }
}

// one thread per (variable, component): rhs = -sum of the factors' b_i / b_j
__global__ void k_assemble_rhs(const gvox_linear_factor* __restrict__ rec,
                               const int32_t* __restrict__ g_start, const int32_t* __restrict__ g_list,
                               int64_t num_vars, double* __restrict__ rhs) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 6 * num_vars) return;
  const int64_t v = t / 6;
  const int e = (int)(t % 6);
  double s = 0.0;
  for (int32_t c = g_start[v]; c < g_start[v + 1]; ++c) {
    const int32_t x = g_list[c];
    const gvox_linear_factor& r = rec[x >> 1];
    s += (x & 1) ? r.b_j[e] : r.b_i[e];
  }
  rhs[t] = -s;
}

// block-Jacobi preconditioner: Minv_v = (diag block)^-1 by Cholesky (fp64)
__global__ void k_block_jacobi(const double* __restrict__ blocks, const int32_t* __restrict__ diag_block,
                               int64_t num_vars, double* __restrict__ minv, int32_t* __restrict__ bad) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= num_vars) return;
  double L[36];
  const double* A = blocks + 36 * (int64_t)diag_block[v];
  for (int i = 0; i < 36; ++i) L[i] = A[i];
  for (int j = 0; j < 6; ++j) {
    double d = L[j * 6 + j];
    for (int k = 0; k < j; ++k) d -= L[j * 6 + k] * L[j * 6 + k];
    if (!(d > 0.0) || !isfinite(d)) {
      atomicOr(bad, 1);
      for (int i = 0; i < 36; ++i) minv[36 * v + i] = (i % 7 == 0) ? 1.0 : 0.0;
      return;
    }
    const double ljj = sqrt(d);
    L[j * 6 + j] = ljj;
    for (int i = j + 1; i < 6; ++i) {
      double s = L[i * 6 + j];
      for (int k = 0; k < j; ++k) s -= L[i * 6 + k] * L[j * 6 + k];
      L[i * 6 + j] = s / ljj;
    }
  }
  // columns of the inverse: solve L L^T x = e_c
  for (int c = 0; c < 6; ++c) {
    double y[6], x[6];
    for (int i = 0; i < 6; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= L[i * 6 + k] * y[k];
      y[i] = s / L[i * 6 + i];
    }
    for (int i = 5; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < 6; ++k) s -= L[k * 6 + i] * x[k];
      x[i] = s / L[i * 6 + i];
    }
    for (int i = 0; i < 6; ++i) minv[36 * v + i * 6 + c] = x[i];
  }
}

// deterministic block-wide sum (fixed strided order, then a fixed tree)
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

__device__ inline void precond(const double* __restrict__ minv, const double* __restrict__ r,
                               double* __restrict__ z, int64_t n6) {
  for (int64_t t = threadIdx.x; t < n6; t += blockDim.x) {
    const int64_t v = t / 6;
    const int i = (int)(t % 6);
    double s = 0.0;
    for (int k = 0; k < 6; ++k) s += minv[36 * v + i * 6 + k] * r[6 * v + k];
    z[t] = s;
  }
}

// PCG start: x = 0, r = rhs, z = M^-1 r, p = z, rz = r.z, r0 = |r|
__global__ void __launch_bounds__(kUpdThreads)
    k_pcg_init(const double* __restrict__ rhs, const double* __restrict__ minv, int64_t num_vars,
               double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
               double* __restrict__ p, PcgState* __restrict__ st) {
  __shared__ double red[33];
  const int64_t n6 = 6 * num_vars;
  for (int64_t t = threadIdx.x; t < n6; t += blockDim.x) {
    x[t] = 0.0;
    r[t] = rhs[t];
  }
  __syncthreads();
  precond(minv, r, z, n6);
  __syncthreads();
  double rz = 0.0, rr = 0.0;
  for (int64_t t = threadIdx.x; t < n6; t += blockDim.x) {
    p[t] = z[t];
    rz += r[t] * z[t];
    rr += r[t] * r[t];
  }
  rz = block_sum(rz, red);
  rr = block_sum(rr, red);
  if (threadIdx.x == 0) {
    st->rz = rz;
    st->r0 = sqrt(rr);
    st->res = sqrt(rr);
    st->iter = 0;
  }
}

// q = A p (one warp per block row; lane l takes the row's blocks l, l + 32, ...
// then a fixed xor tree), and per-row partials of p . q
__global__ void k_spmv_dot(const double* __restrict__ blocks, const int32_t* __restrict__ row_start,
                           const int32_t* __restrict__ col, int64_t num_vars,
                           const double* __restrict__ p, double* __restrict__ q,
                           double* __restrict__ pq_part) {
  const int lane = threadIdx.x & 31;
  const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (v >= num_vars) return;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int32_t b = row_start[v] + lane; b < row_start[v + 1]; b += 32) {
    const double* B = blocks + 36 * (int64_t)b;
    const double* pc = p + 6 * (int64_t)col[b];
    double pv[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) pv[k] = pc[k];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int k = 0; k < 6; ++k) acc[i] += B[i * 6 + k] * pv[k];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 6; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  if (lane == 0) {
    double d = 0.0;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      q[6 * v + i] = acc[i];
      d += p[6 * v + i] * acc[i];
    }
    pq_part[v] = d;
  }
}

// one block: alpha, x, r, z, beta, p; sets the WHILE condition
__global__ void __launch_bounds__(kUpdThreads)
    k_pcg_update(const double* __restrict__ minv, int64_t num_vars, const double* __restrict__ q,
                 const double* __restrict__ pq_part, double* __restrict__ x, double* __restrict__ r,
                 double* __restrict__ z, double* __restrict__ p, PcgState* __restrict__ st,
                 int32_t max_iter, double tol, cudaGraphConditionalHandle cond) {
  __shared__ double red[33];
  const int64_t n6 = 6 * num_vars;
  double pq = 0.0;
  for (int64_t v = threadIdx.x; v < num_vars; v += blockDim.x) pq += pq_part[v];
  pq = block_sum(pq, red);
  const double rz = st->rz;
  const double alpha = pq > 0.0 ? rz / pq : 0.0;
  for (int64_t t = threadIdx.x; t < n6; t += blockDim.x) {
    x[t] += alpha * p[t];
    r[t] -= alpha * q[t];
  }
  __syncthreads();
  precond(minv, r, z, n6);
  __syncthreads();
  double rzn = 0.0, rr = 0.0;
  for (int64_t t = threadIdx.x; t < n6; t += blockDim.x) {
    rzn += r[t] * z[t];
    rr += r[t] * r[t];
  }
  rzn = block_sum(rzn, red);
  rr = block_sum(rr, red);
  const double beta = rz > 0.0 ? rzn / rz : 0.0;
  for (int64_t t = threadIdx.x; t < n6; t += blockDim.x) p[t] = z[t] + beta * p[t];
  if (threadIdx.x == 0) {
    st->rz = rzn;
    st->res = sqrt(rr);
    st->iter += 1;
    const bool go = st->res > tol * st->r0 && st->iter < max_iter && pq > 0.0;
    if (cond) cudaGraphSetConditional(cond, go ? 1u : 0u);
    st->done = go ? 0 : 1;
  }
}

// delta of every pose: the solution for variables, 0 for fixed poses
__global__ void k_scatter_delta(const double* __restrict__ x, const int32_t* __restrict__ var_of_pose,
                                int64_t num_poses, double* __restrict__ delta) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 6 * num_poses) return;
  const int32_t v = var_of_pose[t / 6];
  delta[t] = v >= 0 ? x[6 * (int64_t)v + t % 6] : 0.0;
}

// Persistent PCG: one cooperative launch runs every iteration; three grid
// barriers per iteration (after q = A p; after x, r, z; after p).  Every CTA
// sums the per-row partials itself in the same fixed order, so all CTAs hold
// bitwise identical alpha, beta and stopping decisions (and the run is
// reproducible).  Rows are grid-strided warp by warp.
constexpr int kPcgThreads = 256;

__device__ double sum_parts(const double* __restrict__ part, int64_t n, double* red) {
  double s = 0.0;
  for (int64_t v = threadIdx.x; v < n; v += blockDim.x) s += part[v];
  return block_sum(s, red);
}

// two block sums in one pass (same per-thread order and tree as block_sum)
__device__ void block_sum2(double& a, double& b, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __syncthreads();
  if (lane == 0) {
    red[w] = a;
    red[32 + w] = b;
  }
  __syncthreads();
  if (w == 0) {
    double x = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    double y = lane < (int)(blockDim.x >> 5) ? red[32 + lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      x += __shfl_xor_sync(0xffffffffu, x, o);
      y += __shfl_xor_sync(0xffffffffu, y, o);
    }
    if (lane == 0) {
      red[64] = x;
      red[65] = y;
    }
  }
  __syncthreads();
  a = red[64];
  b = red[65];
}

__global__ void __launch_bounds__(kPcgThreads)
    k_pcg_persistent(const double* __restrict__ blocks, const int32_t* __restrict__ row_start,
                     const int32_t* __restrict__ col, int64_t num_vars, const double* __restrict__ minv,
                     const double* __restrict__ rhs, double* __restrict__ x, double* __restrict__ r,
                     double* __restrict__ z, double* __restrict__ p, double* __restrict__ q,
                     double* __restrict__ part_a, double* __restrict__ part_b, PcgState* __restrict__ st,
                     int32_t max_iter, double tol, const int32_t* __restrict__ chunk_row,
                     const int32_t* __restrict__ chunk_b0, const int32_t* __restrict__ row_chunk,
                     int64_t num_chunks, double* __restrict__ qpart, double* __restrict__ part_c) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[33];
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // z = M^-1 r for the rows of this warp; returns (r.z, r.r) partials per row
  auto precond_rows = [&]() {
    for (int64_t v = gwarp; v < num_vars; v += nwarps) {
      double zi = 0.0, rv = 0.0;
      if (lane < 6) {
        rv = r[6 * v + lane];
        for (int k = 0; k < 6; ++k) zi += minv[36 * v + lane * 6 + k] * r[6 * v + k];
        z[6 * v + lane] = zi;
      }
      double rz = lane < 6 ? rv * zi : 0.0, rr = lane < 6 ? rv * rv : 0.0;
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        rz += __shfl_xor_sync(0xffffffffu, rz, o);
        rr += __shfl_xor_sync(0xffffffffu, rr, o);
      }
      if (lane == 0) {
        part_a[v] = rz;
        part_b[v] = rr;
      }
    }
  };
  // ---- start: x = 0, r = rhs, z = M^-1 r, p = z
  for (int64_t v = gwarp; v < num_vars; v += nwarps)
    if (lane < 6) {
      x[6 * v + lane] = 0.0;
      r[6 * v + lane] = rhs[6 * v + lane];
    }
  __syncwarp();
  precond_rows();
  for (int64_t v = gwarp; v < num_vars; v += nwarps)
    if (lane < 6) p[6 * v + lane] = z[6 * v + lane];
  grid.sync();
  double rz = sum_parts(part_a, num_vars, red);
  const double r0 = sqrt(sum_parts(part_b, num_vars, red));
  double res = r0;
  int32_t it = 0;
  bool go = r0 > 0.0 && !(r0 <= tol * r0);
  while (go) {
    // q = A p over row CHUNKS of at most kPcgChunk blocks (a long block row is
    // split over several warps, so the SpMV phase is not as long as the longest
    // row): warp per chunk, lane-strided blocks, fixed xor tree; the chunk's
    // partial product and its p . (partial q) go to qpart / part_c
    for (int64_t c = gwarp; c < num_chunks; c += nwarps) {
      const int32_t v = chunk_row[c];
      const int32_t bend = (c + 1 < num_chunks && chunk_row[c + 1] == v) ? chunk_b0[c + 1]
                                                                          : row_start[v + 1];
      double acc[6] = {0, 0, 0, 0, 0, 0};
      for (int32_t b = chunk_b0[c] + lane; b < bend; b += 32) {
        const double* B = blocks + 36 * (int64_t)b;
        const double* pc = p + 6 * (int64_t)col[b];
        double pv[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) pv[k] = pc[k];
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
          for (int k = 0; k < 6; ++k) acc[i] += B[i * 6 + k] * pv[k];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < 6; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
      if (lane == 0) {
        double d = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          qpart[6 * c + i] = acc[i];
          d += p[6 * (int64_t)v + i] * acc[i];
        }
        part_c[c] = d;
      }
    }
    grid.sync();
    const double pq = sum_parts(part_c, num_chunks, red);
    const double alpha = pq > 0.0 ? rz / pq : 0.0;
    grid.sync();  // every CTA has read part_c before it is overwritten
    for (int64_t v = gwarp; v < num_vars; v += nwarps)
      if (lane < 6) {
        double qv = 0.0;  // the row's chunks in order
        for (int32_t c = row_chunk[v]; c < row_chunk[v + 1]; ++c) qv += qpart[6 * (int64_t)c + lane];
        q[6 * v + lane] = qv;
        x[6 * v + lane] += alpha * p[6 * v + lane];
        r[6 * v + lane] -= alpha * qv;
      }
    __syncwarp();
    precond_rows();
    grid.sync();
    const double rzn = sum_parts(part_a, num_vars, red);
    res = sqrt(sum_parts(part_b, num_vars, red));
    const double beta = rz > 0.0 ? rzn / rz : 0.0;
    rz = rzn;
    ++it;
    for (int64_t v = gwarp; v < num_vars; v += nwarps)
      if (lane < 6) p[6 * v + lane] = z[6 * v + lane] + beta * p[6 * v + lane];
    go = res > tol * r0 && it < max_iter && pq > 0.0;
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->rz = rz;
    st->r0 = r0;
    st->res = res;
    st->iter = it;
    st->done = 1;
  }
}

// Persistent PCG with TWO grid barriers per iteration (default; the kernel
// above has four).  The direction p = z + beta p is not a phase of its own:
// the SpMV forms p of every column block on the fly, fma(beta, p_old, z) (the
// same expression, so bitwise the value the row's owner stores), and the
// owner writes its rows' p in the update phase after the barrier, when no warp
// reads p_old any more.  Per iteration:
//   phase 1: q partials = A (z + beta p) over row chunks, p . q partials  | grid.sync
//   phase 2: alpha (every CTA sums the chunk partials in the same order);
//            own rows: p, q = sum of the chunks, x += alpha p, r -= alpha q,
//            z = M^-1 r, (r.z, r.r) partials                              | grid.sync
//   phase 3: beta, residual, stopping test (every CTA, same order)
// The chunk partials are rewritten in the next phase 1 only after the second
// barrier, and the row partials in the next phase 2 only after the next first
// barrier, so no buffer needs doubling.  Same PCG recurrence as the 4-barrier
// kernel and the WHILE-node version (rounding may differ in the last bits).
__global__ void __launch_bounds__(kPcgThreads)
    k_pcg_persistent2(const double* __restrict__ blocks, const int32_t* __restrict__ row_start,
                      const int32_t* __restrict__ col, int64_t num_vars, const double* __restrict__ minv,
                      const double* __restrict__ rhs, double* __restrict__ x, double* __restrict__ r,
                      double* __restrict__ z, double* __restrict__ p, double* __restrict__ q,
                      double* __restrict__ part_a, double* __restrict__ part_b, PcgState* __restrict__ st,
                      int32_t max_iter, double tol, const int32_t* __restrict__ chunk_row,
                      const int32_t* __restrict__ chunk_b0, const int32_t* __restrict__ row_chunk,
                      int64_t num_chunks, double* __restrict__ qpart, double* __restrict__ part_c) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[66];
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // z = M^-1 r and the (r.z, r.r) partials of this warp's rows
  auto precond_rows = [&](int64_t v) {
    double zi = 0.0, rv = 0.0;
    if (lane < 6) {
      rv = r[6 * v + lane];
      for (int k = 0; k < 6; ++k) zi += minv[36 * v + lane * 6 + k] * r[6 * v + k];
      z[6 * v + lane] = zi;
    }
    double rz = lane < 6 ? rv * zi : 0.0, rr = lane < 6 ? rv * rv : 0.0;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      rz += __shfl_xor_sync(0xffffffffu, rz, o);
      rr += __shfl_xor_sync(0xffffffffu, rr, o);
    }
    if (lane == 0) {
      part_a[v] = rz;
      part_b[v] = rr;
    }
  };
  // ---- start: x = 0, r = rhs, z = M^-1 r, p = 0 (the first direction is
  // z + 0 * p = z)
  for (int64_t v = gwarp; v < num_vars; v += nwarps) {
    if (lane < 6) {
      x[6 * v + lane] = 0.0;
      r[6 * v + lane] = rhs[6 * v + lane];
      p[6 * v + lane] = 0.0;
    }
    __syncwarp();
    precond_rows(v);
  }
  grid.sync();
  double rz = 0.0, r0 = 0.0;
  for (int64_t v = threadIdx.x; v < num_vars; v += blockDim.x) {
    rz += part_a[v];
    r0 += part_b[v];
  }
  block_sum2(rz, r0, red);
  r0 = sqrt(r0);
  double res = r0, beta = 0.0;
  int32_t it = 0;
  bool go = r0 > 0.0 && !(r0 <= tol * r0);
  while (go) {
    // phase 1: chunk partials of A (z + beta p) and their dot with the row's p
    for (int64_t c = gwarp; c < num_chunks; c += nwarps) {
      const int32_t v = chunk_row[c];
      const int32_t bend = (c + 1 < num_chunks && chunk_row[c + 1] == v) ? chunk_b0[c + 1]
                                                                          : row_start[v + 1];
      double acc[6] = {0, 0, 0, 0, 0, 0};
      for (int32_t b = chunk_b0[c] + lane; b < bend; b += 32) {
        const double* B = blocks + 36 * (int64_t)b;
        const int64_t c6 = 6 * (int64_t)col[b];
        double pv[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) pv[k] = fma(beta, p[c6 + k], z[c6 + k]);
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
          for (int k = 0; k < 6; ++k) acc[i] += B[i * 6 + k] * pv[k];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < 6; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
      if (lane == 0) {
        double d = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          qpart[6 * c + i] = acc[i];
          d += fma(beta, p[6 * (int64_t)v + i], z[6 * (int64_t)v + i]) * acc[i];
        }
        part_c[c] = d;
      }
    }
    grid.sync();
    // phase 2: alpha, then the row updates
    const double pq = sum_parts(part_c, num_chunks, red);
    const double alpha = pq > 0.0 ? rz / pq : 0.0;
    for (int64_t v = gwarp; v < num_vars; v += nwarps) {
      if (lane < 6) {
        const int64_t e = 6 * v + lane;
        const double pv = fma(beta, p[e], z[e]);
        double qv = 0.0;  // the row's chunks in order
        for (int32_t c = row_chunk[v]; c < row_chunk[v + 1]; ++c) qv += qpart[6 * (int64_t)c + lane];
        p[e] = pv;
        q[e] = qv;
        x[e] += alpha * pv;
        r[e] -= alpha * qv;
      }
      __syncwarp();
      precond_rows(v);
    }
    grid.sync();
    // phase 3: beta and the stopping test (identical in every CTA)
    double rzn = 0.0, rr = 0.0;  // (r.z, r.r) in one pass
    for (int64_t v = threadIdx.x; v < num_vars; v += blockDim.x) {
      rzn += part_a[v];
      rr += part_b[v];
    }
    block_sum2(rzn, rr, red);
    res = sqrt(rr);
    beta = rz > 0.0 ? rzn / rz : 0.0;
    rz = rzn;
    ++it;
    go = res > tol * r0 && it < max_iter && pq > 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->rz = rz;
    st->r0 = r0;
    st->res = res;
    st->iter = it;
    st->done = 1;
  }
}

// Cluster PCG (small and medium graphs): the same iteration on ONE thread-block
// cluster of up to 16 CTAs (one per SM) instead of the whole grid.  The three
// barriers per iteration are hardware cluster barriers (barrier.cluster
// arrive.release / wait.acquire: the CTAs' global writes of q, x, r, z, p are
// visible cluster-wide after them) instead of grid-wide software barriers, and
// the dot products are reduced through distributed shared memory: each CTA
// publishes its deterministic block sum in its own shared memory and every CTA
// reads all of them in rank order, so every CTA holds bitwise the same alpha,
// beta and stopping decision.  The SpMV rows are strided over the cluster's
// warps exactly as over the grid's.
__global__ void __launch_bounds__(kPcgThreads)
    k_pcg_cluster(const double* __restrict__ blocks, const int32_t* __restrict__ row_start,
                  const int32_t* __restrict__ col, int64_t num_vars, const double* __restrict__ minv,
                  const double* __restrict__ rhs, double* __restrict__ x, double* __restrict__ r,
                  double* __restrict__ z, double* __restrict__ p, double* __restrict__ q,
                  PcgState* __restrict__ st, int32_t max_iter, double tol) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double red[33];
  __shared__ double cpart[3];  // this CTA's (p.q), (r.z), (r.r)
  const int lane = threadIdx.x & 31;
  const unsigned rank = cluster.block_rank(), nct = cluster.num_blocks();
  const int64_t gwarp = ((int64_t)rank * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)nct * blockDim.x) >> 5;
  // sum of every CTA's slot, in rank order (after a cluster barrier)
  auto cluster_sum = [&](int slot) -> double {
    double s = 0.0;
    for (unsigned c = 0; c < nct; ++c) s += *cluster.map_shared_rank(&cpart[slot], c);
    return s;
  };
  // z = M^-1 r on this warp's rows; (r.z, r.r) of the CTA into cpart[1], cpart[2]
  auto precond_rows = [&]() {
    double rz = 0.0, rr = 0.0;
    for (int64_t v = gwarp; v < num_vars; v += nwarps) {
      double zi = 0.0, rv = 0.0;
      if (lane < 6) {
        rv = r[6 * v + lane];
        for (int k = 0; k < 6; ++k) zi += minv[36 * v + lane * 6 + k] * r[6 * v + k];
        z[6 * v + lane] = zi;
      }
      rz += lane < 6 ? rv * zi : 0.0;
      rr += lane < 6 ? rv * rv : 0.0;
    }
    rz = block_sum(rz, red);
    rr = block_sum(rr, red);
    if (threadIdx.x == 0) {
      cpart[1] = rz;
      cpart[2] = rr;
    }
  };
  for (int64_t v = gwarp; v < num_vars; v += nwarps)
    if (lane < 6) {
      x[6 * v + lane] = 0.0;
      r[6 * v + lane] = rhs[6 * v + lane];
    }
  __syncwarp();
  precond_rows();
  for (int64_t v = gwarp; v < num_vars; v += nwarps)
    if (lane < 6) p[6 * v + lane] = z[6 * v + lane];
  cluster.sync();
  double rz = cluster_sum(1);
  const double r0 = sqrt(cluster_sum(2));
  double res = r0;
  int32_t it = 0;
  bool go = r0 > 0.0 && !(r0 <= tol * r0);
  while (go) {
    // q = A p (warp per block row, lane-strided blocks, fixed xor tree)
    double pqp = 0.0;
    for (int64_t v = gwarp; v < num_vars; v += nwarps) {
      double acc[6] = {0, 0, 0, 0, 0, 0};
      for (int32_t b = row_start[v] + lane; b < row_start[v + 1]; b += 32) {
        const double* B = blocks + 36 * (int64_t)b;
        const double* pc = p + 6 * (int64_t)col[b];
        double pv[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) pv[k] = pc[k];
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
          for (int k = 0; k < 6; ++k) acc[i] += B[i * 6 + k] * pv[k];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < 6; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
      if (lane == 0) {
        double d = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          q[6 * v + i] = acc[i];
          d += p[6 * v + i] * acc[i];
        }
        pqp += d;
      }
    }
    pqp = block_sum(pqp, red);
    if (threadIdx.x == 0) cpart[0] = pqp;
    cluster.sync();  // q and every CTA's p.q published
    const double pq = cluster_sum(0);
    const double alpha = pq > 0.0 ? rz / pq : 0.0;
    for (int64_t v = gwarp; v < num_vars; v += nwarps)
      if (lane < 6) {
        x[6 * v + lane] += alpha * p[6 * v + lane];
        r[6 * v + lane] -= alpha * q[6 * v + lane];
      }
    __syncwarp();
    precond_rows();
    cluster.sync();  // (r.z, r.r) published; every CTA has read p.q
    const double rzn = cluster_sum(1);
    res = sqrt(cluster_sum(2));
    const double beta = rz > 0.0 ? rzn / rz : 0.0;
    rz = rzn;
    ++it;
    for (int64_t v = gwarp; v < num_vars; v += nwarps)
      if (lane < 6) p[6 * v + lane] = z[6 * v + lane] + beta * p[6 * v + lane];
    go = res > tol * r0 && it < max_iter && pq > 0.0;
    cluster.sync();  // p complete; every CTA has read (r.z, r.r)
  }
  if (rank == 0 && threadIdx.x == 0) {
    st->rz = rz;
    st->r0 = r0;
    st->res = res;
    st->iter = it;
    st->done = 1;
  }
}

}  // namespace

// The cluster PCG when the matrix is at most GVOX_PCG_CLUSTER_MB MB of blocks
// (default 0: never).  Measured on C4 (500 poses, 47k blocks, r02k): 12.9 ms
// against 7.2 ms for the grid-wide persistent kernel -- the cheaper barriers
// do not pay for 16 CTAs' worth of SpMV warps (each walks ~4 block rows in
// sequence; long_scoreboard 19.8 cycles/issue), so the grid kernel stays the
// default.  Returns false (nothing launched) when not selected or when no
// cluster of 16 or 8 CTAs can be launched; the caller then runs the grid kernel.
bool launch_pcg_cluster(const double* blocks, const int32_t* row_start, const int32_t* col,
                        int64_t num_vars, int64_t num_blocks, const double* minv, const double* rhs,
                        double* x, double* r, double* z, double* p, double* q, PcgState* st,
                        int32_t max_iter, double tol, cudaStream_t stream) {
  double limit_mb = 0.0;
  if (const char* e = std::getenv("GVOX_PCG_CLUSTER_MB")) limit_mb = std::atof(e);
  if (limit_mb <= 0.0 || (double)num_blocks * 288.0 > limit_mb * 1048576.0) return false;
  cudaFuncSetAttribute(k_pcg_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c : {16, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)c);
    cfg.blockDim = dim3(kPcgThreads);
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, (void*)k_pcg_cluster, &cfg) != cudaSuccess ||
        nclusters < 1) {
      cudaGetLastError();
      continue;
    }
    if (cudaLaunchKernelEx(&cfg, k_pcg_cluster, blocks, row_start, col, num_vars, minv, rhs, x, r,
                           z, p, q, st, max_iter, tol) == cudaSuccess) {
      note_launch();
      return true;
    }
    cudaGetLastError();
  }
  return false;
}

void launch_pcg_persistent(const double* blocks, const int32_t* row_start, const int32_t* col,
                           int64_t num_vars, const double* minv, const double* rhs, double* x,
                           double* r, double* z, double* p, double* q, double* part_a,
                           double* part_b, PcgState* st, int32_t max_iter, double tol,
                           const int32_t* chunk_row, const int32_t* chunk_b0,
                           const int32_t* row_chunk, int64_t num_chunks, double* qpart,
                           double* part_c, cudaStream_t stream) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // two grid barriers per iteration (default) or four (GVOX_PCG_BARRIERS=4)
  const char* eb = std::getenv("GVOX_PCG_BARRIERS");
  void* kern = (eb && std::atoi(eb) == 4) ? (void*)k_pcg_persistent : (void*)k_pcg_persistent2;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPcgThreads, 0);
  const int64_t want = (std::max(num_vars, num_chunks) * 32 + kPcgThreads - 1) / kPcgThreads;  // a warp per chunk
  int grid = (int)std::min<int64_t>(std::max<int64_t>(want, 1), (int64_t)sms * std::max(per_sm, 1));
  if (const char* e = std::getenv("GVOX_PCG_CTAS"))  // experiments: fewer, busier CTAs
    grid = std::max(1, std::min(grid, std::atoi(e)));
  void* args[] = {(void*)&blocks, (void*)&row_start, (void*)&col, (void*)&num_vars, (void*)&minv,
                  (void*)&rhs, (void*)&x, (void*)&r, (void*)&z, (void*)&p, (void*)&q,
                  (void*)&part_a, (void*)&part_b, (void*)&st, (void*)&max_iter, (void*)&tol,
                  (void*)&chunk_row, (void*)&chunk_b0, (void*)&row_chunk, (void*)&num_chunks,
                  (void*)&qpart, (void*)&part_c};
  cudaLaunchCooperativeKernel(kern, grid, kPcgThreads, args, 0, stream);
  note_launch();
}

void launch_assemble(const gvox_linear_factor* rec, const int32_t* contrib_start,
                     const int32_t* contrib, int64_t num_blocks, const uint8_t* is_diag,
                     double lambda, double* blocks, const int32_t* g_start, const int32_t* g_list,
                     int64_t num_vars, double* rhs, const int32_t* diag_block, double* minv,
                     int32_t* bad, cudaStream_t stream) {
  if (num_blocks > 0) {
    k_assemble_blocks<<<(unsigned)((num_blocks * 32 + 255) / 256), 256, 0, stream>>>(
        rec, contrib_start, contrib, num_blocks, is_diag, lambda, blocks);
    note_launch();
  }
  if (num_vars > 0) {
    k_assemble_rhs<<<(unsigned)((6 * num_vars + 255) / 256), 256, 0, stream>>>(rec, g_start, g_list,
                                                                              num_vars, rhs);
    k_block_jacobi<<<(unsigned)((num_vars + 127) / 128), 128, 0, stream>>>(blocks, diag_block, num_vars,
                                                                          minv, bad);
    note_launch();
    note_launch();
  }
}

void launch_pcg_init(const double* rhs, const double* minv, int64_t num_vars, double* x, double* r,
                     double* z, double* p, PcgState* st, cudaStream_t stream) {
  k_pcg_init<<<1, kUpdThreads, 0, stream>>>(rhs, minv, num_vars, x, r, z, p, st);
  note_launch();
}

void launch_pcg_iteration(const double* blocks, const int32_t* row_start, const int32_t* col,
                          int64_t num_vars, const double* minv, double* x, double* r, double* z,
                          double* p, double* q, double* pq_part, PcgState* st, int32_t max_iter,
                          double tol, cudaGraphConditionalHandle cond, cudaStream_t stream) {
  k_spmv_dot<<<(unsigned)((num_vars * 32 + 255) / 256), 256, 0, stream>>>(blocks, row_start, col,
                                                                          num_vars, p, q, pq_part);
  k_pcg_update<<<1, kUpdThreads, 0, stream>>>(minv, num_vars, q, pq_part, x, r, z, p, st, max_iter,
                                              tol, cond);
  note_launch();
  note_launch();
}

void launch_scatter_delta(const double* x, const int32_t* var_of_pose, int64_t num_poses,
                          double* delta, cudaStream_t stream) {
  if (num_poses <= 0) return;
  k_scatter_delta<<<(unsigned)((6 * num_poses + 255) / 256), 256, 0, stream>>>(x, var_of_pose,
                                                                              num_poses, delta);
  note_launch();
}

}  // namespace gvox
