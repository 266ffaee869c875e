// k_register.cu -- the solve/update step of the on-device registration loop
// (gvox_register_batch, include/gvox.h).  One loop
// iteration is k_linearize -> k_reduce (compact records) -> k_gn_step, the
// body of a CUDA graph WHILE node; k_gn_step sets the node's condition.
//
// Per variable pose v (a "problem"), one warp:
//   H = sum_f H_ii(f), b = sum_f b_i(f), e = sum_f e(f) over v's factors (lane
//   l takes factors l, l + 32, ...; then a fixed xor-tree sum over lanes, so
//   the result depends only on the problem's factor list), with H_ii = Ad^T H_jj Ad and b_i = -Ad^T b_j
//   (Ad = Ad(T_ij); exact since A = -B Ad(T_ij), Eqs. 4-8);
//   (H + lambda I) delta = -b by fp64 Cholesky; T_v <- T_v Exp(delta).
#include <cuda_runtime.h>

#include "k_common.cuh"

namespace gvox {
namespace {

constexpr int kStepWarps = 8;

// Ad(T) for rotation-first tangents: [[R, 0], [t^ R, R]] (row-major 6x6).
__device__ inline void adjoint6_r(const double* R, const double* t, double* Ad) {
  for (int i = 0; i < 36; ++i) Ad[i] = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      Ad[a * 6 + b] = R[a * 3 + b];
      Ad[(a + 3) * 6 + (b + 3)] = R[a * 3 + b];
    }
  const double T[9] = {0, -t[2], t[1], t[2], 0, -t[0], -t[1], t[0], 0};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double s = 0;
      for (int c = 0; c < 3; ++c) s += T[a * 3 + c] * R[c * 3 + b];
      Ad[(a + 3) * 6 + b] = s;
    }
}

// SE(3) exponential, rotation-first xi = [w; rho]:
//   R = I + A K + B K^2,  t = (I + B K + C K^2) rho,  K = w^,
//   A = sin(th)/th, B = (1 - cos th)/th^2, C = (th - sin th)/th^3.
__device__ inline void se3_exp_dev(const double* xi, double* R, double* t) {
  const double w0 = xi[0], w1 = xi[1], w2 = xi[2];
  const double th2 = w0 * w0 + w1 * w1 + w2 * w2;
  const double th = sqrt(th2);
  double A, B, C;
  if (th < 1e-4) {  // series; the truncation error is below 1e-17
    A = 1.0 - th2 / 6.0 + th2 * th2 / 120.0;
    B = 0.5 - th2 / 24.0 + th2 * th2 / 720.0;
    C = 1.0 / 6.0 - th2 / 120.0 + th2 * th2 / 5040.0;
  } else {
    double s, c;
    sincos(th, &s, &c);
    A = s / th;
    B = (1.0 - c) / th2;
    C = (th - s) / (th2 * th);
  }
  const double K[9] = {0, -w2, w1, w2, 0, -w0, -w1, w0, 0};
  double K2[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double s = 0;
      for (int c = 0; c < 3; ++c) s += K[a * 3 + c] * K[c * 3 + b];
      K2[a * 3 + b] = s;
    }
  double V[9];
  for (int i = 0; i < 9; ++i) {
    const double I = (i % 4 == 0) ? 1.0 : 0.0;
    R[i] = I + A * K[i] + B * K2[i];
    V[i] = I + B * K[i] + C * K2[i];
  }
  for (int a = 0; a < 3; ++a) t[a] = V[a * 3 + 0] * xi[3] + V[a * 3 + 1] * xi[4] + V[a * 3 + 2] * xi[5];
}

// In-place Cholesky of a 6x6 SPD matrix (row-major, lower factor) and solve
// L L^T x = rhs.  False if a pivot is not positive and finite.
__device__ inline bool chol6_solve(double* M, const double* rhs, double* x) {
  for (int j = 0; j < 6; ++j) {
    double d = M[j * 6 + j];
    for (int k = 0; k < j; ++k) d -= M[j * 6 + k] * M[j * 6 + k];
    if (!(d > 0.0) || !isfinite(d)) return false;
    const double ljj = sqrt(d);
    M[j * 6 + j] = ljj;
    for (int i = j + 1; i < 6; ++i) {
      double s = M[i * 6 + j];
      for (int k = 0; k < j; ++k) s -= M[i * 6 + k] * M[j * 6 + k];
      M[i * 6 + j] = s / ljj;
    }
  }
  double y[6];
  for (int i = 0; i < 6; ++i) {
    double s = rhs[i];
    for (int k = 0; k < i; ++k) s -= M[i * 6 + k] * y[k];
    y[i] = s / M[i * 6 + i];
  }
  for (int i = 5; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < 6; ++k) s -= M[k * 6 + i] * x[k];
    x[i] = s / M[i * 6 + i];
  }
  return true;
}

__global__ void __launch_bounds__(32 * kStepWarps)
    k_gn_step(const RegProblem* __restrict__ problems, int32_t num_problems,
              const int32_t* __restrict__ reg_factors, const FactorDev* __restrict__ factors,
              const gvox_factor_accum* __restrict__ accum, double* __restrict__ poses,
              gvox_register_result* __restrict__ results, int32_t* __restrict__ active,
              RegControl* __restrict__ ctrl, double* __restrict__ history, int64_t num_poses,
              cudaGraphConditionalHandle cond) {
  __shared__ double Ti_s[kStepWarps][12];
  __shared__ double H_s[kStepWarps][36];
  __shared__ double b_s[kStepWarps][6];
  __shared__ int32_t still_active;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) still_active = 0;
  __syncthreads();
  const int32_t iter = ctrl->iter;
  const int32_t p = blockIdx.x * kStepWarps + w;
  if (p < num_problems && active[p]) {
    const RegProblem pr = problems[p];
    const int32_t v = pr.pose;
    if (lane < 12) Ti_s[w][lane] = poses[12 * (int64_t)v + lane];
    __syncwarp();
    // lane l expands the factors pr.f0 + l, pr.f0 + l + 32, ... (H_ii = Ad^T H_jj Ad,
    // b_i = -Ad^T b_j, upper triangle); then a fixed xor-tree sum over lanes
    double hs[21], bs[6], err = 0.0;
    int32_t inl = 0;
#pragma unroll
    for (int i = 0; i < 21; ++i) hs[i] = 0.0;
#pragma unroll
    for (int i = 0; i < 6; ++i) bs[i] = 0.0;
    for (int32_t q = pr.f0 + lane; q < pr.f1; q += 32) {
      const int32_t f = reg_factors[q];
      const FactorDev fd = factors[f];
      const gvox_factor_accum* a = accum + f;
      double Tj[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) Tj[i] = poses[12 * (int64_t)fd.pj + i];
      double R[9], t[3], vv[3], Ad[36], Hj[36];
      relative_pose_dev(Ti_s[w], Tj, R, t, vv);
      adjoint6_r(R, t, Ad);
      int k = 0;
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = r; c < 6; ++c) {
          const double x = a->terms[k++];
          Hj[r * 6 + c] = x;
          Hj[c * 6 + r] = x;
        }
      double M[36];  // H_jj Ad
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          double s2 = 0;
#pragma unroll
          for (int j = 0; j < 6; ++j) s2 += Hj[r * 6 + j] * Ad[j * 6 + c];
          M[r * 6 + c] = s2;
        }
      k = 0;
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = r; c < 6; ++c) {
          double s2 = 0;
#pragma unroll
          for (int j = 0; j < 6; ++j) s2 += Ad[j * 6 + r] * M[j * 6 + c];
          hs[k++] += s2;
        }
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        double s2 = 0;
#pragma unroll
        for (int j = 0; j < 6; ++j) s2 += Ad[j * 6 + c] * a->terms[21 + j];
        bs[c] -= s2;
      }
      err += a->terms[27];
#pragma unroll
      for (int l = 0; l < GVOX_MAX_LEVELS; ++l) inl += a->inliers[l];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int i = 0; i < 21; ++i) hs[i] += __shfl_xor_sync(0xffffffffu, hs[i], o);
#pragma unroll
      for (int i = 0; i < 6; ++i) bs[i] += __shfl_xor_sync(0xffffffffu, bs[i], o);
      err += __shfl_xor_sync(0xffffffffu, err, o);
      inl += __shfl_xor_sync(0xffffffffu, inl, o);
    }
    if (lane == 0) {
      int k = 0;
      for (int r = 0; r < 6; ++r)
        for (int c = r; c < 6; ++c) {
          H_s[w][r * 6 + c] = hs[k];
          H_s[w][c * 6 + r] = hs[k];
          ++k;
        }
      for (int i = 0; i < 6; ++i) b_s[w][i] = bs[i];
    }
    __syncwarp();
    if (lane == 0) {
      gvox_register_result& res = results[v];
      if (iter == 0) res.error_initial = err;
      res.error_final = err;
      res.inliers = inl;
      res.iterations = iter + 1;
      if (history) history[(int64_t)iter * num_poses + v] = err;
      double Mx[36], rhs[6], delta[6];
      for (int e = 0; e < 36; ++e) Mx[e] = H_s[w][e] + ((e % 7 == 0) ? ctrl->lambda : 0.0);
      for (int i = 0; i < 6; ++i) rhs[i] = -b_s[w][i];
      bool go = true;
      if (!chol6_solve(Mx, rhs, delta)) {
        res.status = GVOX_REG_SINGULAR;
        for (int i = 0; i < 6; ++i) res.last_step[i] = 0.0;
        go = false;
      } else {
        double dR[9], dt[3];
        se3_exp_dev(delta, dR, dt);
        const double* T = Ti_s[w];
        double Tn[12];
        for (int a = 0; a < 3; ++a) {
          for (int b = 0; b < 3; ++b)
            Tn[a * 4 + b] = T[a * 4 + 0] * dR[0 * 3 + b] + T[a * 4 + 1] * dR[1 * 3 + b] +
                            T[a * 4 + 2] * dR[2 * 3 + b];
          Tn[a * 4 + 3] = T[a * 4 + 0] * dt[0] + T[a * 4 + 1] * dt[1] + T[a * 4 + 2] * dt[2] + T[a * 4 + 3];
        }
        for (int i = 0; i < 12; ++i) poses[12 * (int64_t)v + i] = Tn[i];
        for (int i = 0; i < 6; ++i) res.last_step[i] = delta[i];
        const double nw = sqrt(delta[0] * delta[0] + delta[1] * delta[1] + delta[2] * delta[2]);
        const double nr = sqrt(delta[3] * delta[3] + delta[4] * delta[4] + delta[5] * delta[5]);
        if (nw <= ctrl->eps_rot && nr <= ctrl->eps_trans) {
          res.status = GVOX_REG_CONVERGED;
          go = false;
        } else if (iter + 1 >= ctrl->max_iter) {
          res.status = GVOX_REG_MAX_ITER;
          go = false;
        }
      }
      if (!go) active[p] = 0;
      else atomicAdd(&still_active, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (still_active) atomicAdd(&ctrl->any_active, still_active);
    __threadfence();
    const unsigned ticket = atomicAdd(&ctrl->blocks_done, 1u);
    if (ticket == gridDim.x - 1) {  // last block: all counts are in
      __threadfence();
      const int32_t any = atomicAdd(&ctrl->any_active, 0);
      ctrl->any_active = 0;
      ctrl->blocks_done = 0;
      ctrl->iter = iter + 1;
      if (cond) cudaGraphSetConditional(cond, any > 0 ? 1u : 0u);  // 0: eager (profiling) mode
    }
  }
}

// Global loop helpers (gvox_optimize_global): T_v <- T_v Exp(delta_v) for every
// pose (fixed poses carry delta = 0: Exp(0) = I leaves them bit-identical),
// and the largest |w| and |rho| of the step; one block, fixed-order maxima.
__global__ void __launch_bounds__(256)
    k_apply_delta(double* __restrict__ poses, const double* __restrict__ delta, int64_t num_poses,
                  double* __restrict__ out_max) {
  __shared__ double mw[256], mr[256];
  double aw = 0.0, ar = 0.0;
  for (int64_t v = threadIdx.x; v < num_poses; v += blockDim.x) {
    const double* d = delta + 6 * v;
    aw = fmax(aw, sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]));
    ar = fmax(ar, sqrt(d[3] * d[3] + d[4] * d[4] + d[5] * d[5]));
    double dR[9], dt[3], T[12];
    se3_exp_dev(d, dR, dt);
    for (int i = 0; i < 12; ++i) T[i] = poses[12 * v + i];
    for (int a = 0; a < 3; ++a) {
      for (int b = 0; b < 3; ++b)
        poses[12 * v + a * 4 + b] = T[a * 4 + 0] * dR[0 * 3 + b] + T[a * 4 + 1] * dR[1 * 3 + b] +
                                    T[a * 4 + 2] * dR[2 * 3 + b];
      poses[12 * v + a * 4 + 3] = T[a * 4 + 0] * dt[0] + T[a * 4 + 1] * dt[1] + T[a * 4 + 2] * dt[2] + T[a * 4 + 3];
    }
  }
  mw[threadIdx.x] = aw;
  mr[threadIdx.x] = ar;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      mw[threadIdx.x] = fmax(mw[threadIdx.x], mw[threadIdx.x + o]);
      mr[threadIdx.x] = fmax(mr[threadIdx.x], mr[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out_max[0] = mw[0];
    out_max[1] = mr[0];
  }
}

// total error of a batch of compact records, fixed order (one block)
__global__ void __launch_bounds__(256)
    k_sum_error(const gvox_factor_accum* __restrict__ acc, int64_t n, double* __restrict__ out) {
  __shared__ double part[256];
  double s = 0.0;
  for (int64_t f = threadIdx.x; f < n; f += blockDim.x) s += acc[f].terms[27];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) part[threadIdx.x] += part[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0];
}

}  // namespace

void launch_apply_delta(double* poses, const double* delta, int64_t num_poses, double* out_max,
                        cudaStream_t stream) {
  k_apply_delta<<<1, 256, 0, stream>>>(poses, delta, num_poses, out_max);
  note_launch();
}

void launch_sum_error(const gvox_factor_accum* acc, int64_t n, double* out, cudaStream_t stream) {
  k_sum_error<<<1, 256, 0, stream>>>(acc, n, out);
  note_launch();
}

void launch_gn_step(const RegProblem* problems, int32_t num_problems, const int32_t* reg_factors,
                    const FactorDev* factors, const gvox_factor_accum* accum, double* poses,
                    gvox_register_result* results, int32_t* active, RegControl* ctrl,
                    double* history, int64_t num_poses, cudaGraphConditionalHandle cond,
                    cudaStream_t stream) {
  const unsigned blocks = (unsigned)((num_problems + kStepWarps - 1) / kStepWarps);
  k_gn_step<<<blocks, 32 * kStepWarps, 0, stream>>>(problems, num_problems, reg_factors, factors,
                                                     accum, poses, results, active, ctrl, history,
                                                     num_poses, cond);
  note_launch();
}

}  // namespace gvox
