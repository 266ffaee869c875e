// k_linearize.cu -- correspondence search + linearization (K3) and the
// per-factor reduction / block expansion (K4).
//
// Paper: Eq.2 e^PC = sum_levels sum_k e^D2D; Eq.3
// e^D2D = d^T (C~ + T_ij C_k T_ij^T)^-1 d with Omega fixed at the
// linearization point; Eqs.4-8 A_k = [R (mu)x, -R],
// B_k = [-(T_ij mu)x, I], H and b sums; P:197 validation and containing-voxel
// lookup; P:221-224 batched linearization.
//
// B200 design ("K4"):
//  * one CTA per tile of TILE consecutive points of one factor; tile -> factor
//    via a device-built table; per-factor constants staged in shared memory.
//  * per point: three coalesced float4 loads (48 B), fp64 transform with the
//    pinned fma order and fp64 key (bit-exact correspondences, reading Q10),
//    fp32 R C R^T once, then per level: hash probe (16 B slot), 48 B voxel
//    gather, fp32 fused covariance, symmetric adjugate inverse, residual
//    d = fp32(centre - q64) + fp32 offset (reading Q12), and the 28 target-block
//    terms of B^T Omega B, B^T Omega d, d^T Omega d accumulated in fp32 per
//    thread.  No tensor cores: the work is 3x3 algebra, not a contraction.
//  * end of tile: fp64 warp-shuffle + shared-memory reduction -> one fp64
//    partial per tile.  K4 sums a factor's tiles in tile order (deterministic)
//    and expands the target block into the paper's blocks with the exact
//    identities H_ii = Ad^T H_jj Ad, H_ij = -Ad^T H_jj, b_i = -Ad^T b_j.
//
// Internal term order (per thread, then per tile):
//   t[0..5]   sum Omega             (xx xy xz yy yz zz)       -> H_tt
//   t[6..14]  sum W, W = Omega [q]x (row-major 3x3)           -> H_tr = -W, H_rt = -W^T
//   t[15..20] sum -[q]x W           (xx xy xz yy yz zz)       -> H_rr
//   t[21..23] sum q x g, g = Omega d                           -> b_rot
//   t[24..26] sum g                                            -> b_trans
//   t[27]     sum d^T g                                        -> error
#include <cstdint>

#include "k_common.cuh"

namespace gvox {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct FactorShared {
  double R[9];
  double t[3];
  double v[3];
  float Rf[9];
  const float4* A;
  const float4* B;
  const float4* N;
  int64_t begin, end;
  int64_t corr_base;
  double r0, inv_r0;
  int L, dyadic, validate, error_only;
  MapLevelDev lv[GVOX_MAX_LEVELS];
};

__global__ void k_tile_map(const int32_t* __restrict__ tile_start, int64_t num_factors,
                           int32_t* __restrict__ tile_factor) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= num_factors) return;
  for (int32_t t = tile_start[f]; t < tile_start[f + 1]; ++t) tile_factor[t] = (int32_t)f;
}

template <int MAXL, bool ALL_DENSE>
__global__ void __launch_bounds__(kThreads, 2)
    k_linearize(const CloudDev* const* __restrict__ clouds, const MapDev* const* __restrict__ maps,
                const FactorDev* __restrict__ factors, const int32_t* __restrict__ tile_start,
                const int32_t* __restrict__ tile_factor, int tile_pts,
                const double* __restrict__ poses, double* __restrict__ partials,
                int64_t* __restrict__ corr) {
  __shared__ FactorShared sh;
  __shared__ double red[kWarps][kPartialStride];
  __shared__ double pose_s[24];

  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;
  // ---- prologue: stage the factor's constants in shared memory
  {
    const int32_t f = __ldg(tile_factor + tile);
    const FactorDev fd = factors[f];
    if (tid < 24) {
      pose_s[tid] = __ldg(poses + 12 * (int64_t)(tid < 12 ? fd.pi : fd.pj) + (tid % 12));
    } else if (tid == 32) {
      const CloudDev* cd = clouds[fd.src];
      int64_t b = (int64_t)(tile - __ldg(tile_start + f)) * tile_pts;
      int64_t e = b + tile_pts;
      int64_t n = cd->n;
      sh.A = cd->A;
      sh.B = cd->B;
      sh.N = cd->N;
      sh.begin = b;
      sh.end = e < n ? e : n;
      sh.validate = (fd.flags & GVOX_F_VALIDATE_SURFACE) && cd->has_normals;
      sh.error_only = (fd.flags & GVOX_F_ERROR_ONLY) ? 1 : 0;
      sh.corr_base = fd.corr_offset;
    } else if (tid == 64) {
      const MapDev* md = maps[fd.tgt];
      sh.L = md->levels;
      sh.dyadic = md->dyadic;
      sh.r0 = md->r0;
      sh.inv_r0 = md->inv_r0;
    } else if (tid >= 96 && tid < 96 + MAXL) {
      const MapDev* md = maps[fd.tgt];
      sh.lv[tid - 96] = md->lv[tid - 96];
    }
    __syncthreads();
    if (tid == 0) {
      relative_pose_dev(pose_s, pose_s + 12, sh.R, sh.t, sh.v);
#pragma unroll
      for (int j = 0; j < 9; ++j) sh.Rf[j] = (float)sh.R[j];
    }
    __syncthreads();
  }

  const int L = sh.L;
  const int dyadic = sh.dyadic;
  const double r0 = sh.r0, inv_r0 = sh.inv_r0;
  const float r0f = (float)sh.r0;
  const bool validate = sh.validate;
  const bool error_only = sh.error_only;
  const int64_t begin = sh.begin, end = sh.end;
  const float4* __restrict__ Ap = sh.A;
  const float4* __restrict__ Bp = sh.B;
  const float4* __restrict__ Np = sh.N;

  float acc[kNumTerms];
#pragma unroll
  for (int j = 0; j < kNumTerms; ++j) acc[j] = 0.f;
  int inl[MAXL];
#pragma unroll
  for (int l = 0; l < MAXL; ++l) inl[l] = 0;
  int n_invisible = 0, n_degenerate = 0;

  // software pipeline: the next point's 48 B source record is in flight while
  // the current one is processed
  float4 na, nb, nc;
  if (begin + tid < end) {
    na = __ldg(Ap + begin + tid);
    nb = __ldg(Bp + begin + tid);
    nc = __ldg(Np + begin + tid);
  }
  for (int64_t k = begin + tid; k < end; k += kThreads) {
    const float4 a = na, b = nb, c = nc;
    if (k + kThreads < end) {
      na = __ldg(Ap + k + kThreads);
      nb = __ldg(Bp + k + kThreads);
      nc = __ldg(Np + k + kThreads);
    }
    const double mx = a.x, my = a.y, mz = a.z;
    if (validate) {
      // discard if (mu - T_i^-1 t_j) . n > 0; zero normal = no test (Q7)
      if (c.y != 0.f || c.z != 0.f || c.w != 0.f) {
        double dx = mx - sh.v[0], dy = my - sh.v[1], dz = mz - sh.v[2];
        double dot = __fma_rn(dx, (double)c.y, __fma_rn(dy, (double)c.z, __dmul_rn(dz, (double)c.w)));
        if (dot > 0.0) {
          ++n_invisible;
          if (corr) {
            for (int l = 0; l < L; ++l) corr[sh.corr_base + k * L + l] = -2;
          }
          continue;
        }
      }
    }
    // q = T_ij mu in fp64, pinned order (Q10)
    const double qx = __fma_rn(sh.R[0], mx, __fma_rn(sh.R[1], my, __fma_rn(sh.R[2], mz, sh.t[0])));
    const double qy = __fma_rn(sh.R[3], mx, __fma_rn(sh.R[4], my, __fma_rn(sh.R[5], mz, sh.t[1])));
    const double qz = __fma_rn(sh.R[6], mx, __fma_rn(sh.R[7], my, __fma_rn(sh.R[8], mz, sh.t[2])));
    const int32_t k0x = clamp_coord(voxel_coord0(qx, r0, inv_r0, dyadic));
    const int32_t k0y = clamp_coord(voxel_coord0(qy, r0, inv_r0, dyadic));
    const int32_t k0z = clamp_coord(voxel_coord0(qz, r0, inv_r0, dyadic));

    const float fqx = (float)qx, fqy = (float)qy, fqz = (float)qz;
    // position inside the level-0 voxel (exact k0 * r0 for dyadic r0)
    const float fx = (float)(qx - (double)k0x * r0);
    const float fy = (float)(qy - (double)k0y * r0);
    const float fz = (float)(qz - (double)k0z * r0);
    bool have_rcr = false;
    float s00 = 0.f, s01 = 0.f, s02 = 0.f, s11 = 0.f, s12 = 0.f, s22 = 0.f;
    // levels are processed in groups of G (all loads of a group in flight together)
    constexpr int G = MAXL < 4 ? MAXL : 4;
#pragma unroll
    for (int lb = 0; lb < MAXL; lb += G) {
      if (lb >= L) break;
      // stage 1: the voxel index of every level of the group
      int32_t vid[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int l = lb + j;
        vid[j] = l < L ? lookup_level<ALL_DENSE>(sh.lv[l], k0x >> l, k0y >> l, k0z >> l) : -1;
      }
      if (corr) {
        for (int j = 0; j < G && lb + j < L; ++j) {
          const int l = lb + j;
          corr[sh.corr_base + k * L + l] =
              vid[j] >= 0 ? (int64_t)pack_key(k0x >> l, k0y >> l, k0z >> l) : -1;
        }
      }
      bool any = false;
#pragma unroll
      for (int j = 0; j < G; ++j) any |= vid[j] >= 0;
      if (!any) continue;

      // stage 2: gather the hit voxels' records (48 B each)
      float4 v0[G], v1[G];
      float v2[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        if (vid[j] >= 0) {
          const float4* vp = sh.lv[lb + j].vox + 3 * (int64_t)vid[j];
          v0[j] = __ldg(vp);
          v1[j] = __ldg(vp + 1);
          v2[j] = __ldg(&vp[2].x);
        }
      }

      // R C R^T in fp32 (symmetric), once per point, overlapping the gathers
      if (!have_rcr) {
        have_rcr = true;
        const float* R = sh.Rf;
        const float m00 = R[0] * a.w + R[1] * b.x + R[2] * b.y;
        const float m01 = R[0] * b.x + R[1] * b.z + R[2] * b.w;
        const float m02 = R[0] * b.y + R[1] * b.w + R[2] * c.x;
        const float m10 = R[3] * a.w + R[4] * b.x + R[5] * b.y;
        const float m11 = R[3] * b.x + R[4] * b.z + R[5] * b.w;
        const float m12 = R[3] * b.y + R[4] * b.w + R[5] * c.x;
        const float m20 = R[6] * a.w + R[7] * b.x + R[8] * b.y;
        const float m21 = R[6] * b.x + R[7] * b.z + R[8] * b.w;
        const float m22 = R[6] * b.y + R[7] * b.w + R[8] * c.x;
        s00 = m00 * R[0] + m01 * R[1] + m02 * R[2];
        s01 = m00 * R[3] + m01 * R[4] + m02 * R[5];
        s02 = m00 * R[6] + m01 * R[7] + m02 * R[8];
        s11 = m10 * R[3] + m11 * R[4] + m12 * R[5];
        s12 = m10 * R[6] + m11 * R[7] + m12 * R[8];
        s22 = m20 * R[6] + m21 * R[7] + m22 * R[8];
      }

      // stage 3: per-level algebra
#pragma unroll
      for (int j = 0; j < G; ++j) {
        if (vid[j] < 0) continue;
        const int l = lb + j;
        // fused covariance (Eq.3) and its inverse by the symmetric adjugate
        const float ca = v0[j].w + s00, cb = v1[j].x + s01, cc = v1[j].y + s02;
        const float cd = v1[j].z + s11, ce = v1[j].w + s12, cf = v2[j] + s22;
        const float i00 = cd * cf - ce * ce;
        const float i01 = cc * ce - cb * cf;
        const float i02 = cb * ce - cc * cd;
        const float i11 = ca * cf - cc * cc;
        const float i12 = cb * cc - ca * ce;
        const float i22 = ca * cd - cb * cb;
        const float det = ca * i00 + cb * i01 + cc * i02;
        // Q16: a fused covariance that is not positive definite contributes nothing
        const bool ok = det > 0.f && det < INFINITY;
        const float id = ok ? __fdividef(1.0f, det) : 0.f;
        n_degenerate += !ok;
        inl[l] += ok;
        const float o00 = i00 * id, o01 = i01 * id, o02 = i02 * id;
        const float o11 = i11 * id, o12 = i12 * id, o22 = i22 * id;

        // d = mu~ - q = (centre_l - q) + offset (Q12).  With f = q - k0 r0 (the
        // point's position inside its level-0 voxel, fp64 -> fp32 once per
        // point) and k_l = k0 >> l:  centre_l - q = r0 (2^(l-1) - (k0 & (2^l - 1))) - f.
        const int mlo = (1 << l) - 1;
        const float hl = 0.5f * (float)(1 << l);
        const float dx = r0f * (hl - (float)(k0x & mlo)) - fx + v0[j].x;
        const float dy = r0f * (hl - (float)(k0y & mlo)) - fy + v0[j].y;
        const float dz = r0f * (hl - (float)(k0z & mlo)) - fz + v0[j].z;

        // g = Omega d, e = d^T g
        const float gx = o00 * dx + o01 * dy + o02 * dz;
        const float gy = o01 * dx + o11 * dy + o12 * dz;
        const float gz = o02 * dx + o12 * dy + o22 * dz;
        acc[27] += dx * gx + dy * gy + dz * gz;
        if (error_only) continue;

        acc[24] += gx;
        acc[25] += gy;
        acc[26] += gz;
        // b_rot = q x g
        acc[21] += fqy * gz - fqz * gy;
        acc[22] += fqz * gx - fqx * gz;
        acc[23] += fqx * gy - fqy * gx;
        // sum Omega
        acc[0] += o00; acc[1] += o01; acc[2] += o02;
        acc[3] += o11; acc[4] += o12; acc[5] += o22;
        // W = Omega [q]x
        const float w00 = o01 * fqz - o02 * fqy, w01 = o02 * fqx - o00 * fqz, w02 = o00 * fqy - o01 * fqx;
        const float w10 = o11 * fqz - o12 * fqy, w11 = o12 * fqx - o01 * fqz, w12 = o01 * fqy - o11 * fqx;
        const float w20 = o12 * fqz - o22 * fqy, w21 = o22 * fqx - o02 * fqz, w22 = o02 * fqy - o12 * fqx;
        acc[6] += w00; acc[7] += w01; acc[8] += w02;
        acc[9] += w10; acc[10] += w11; acc[11] += w12;
        acc[12] += w20; acc[13] += w21; acc[14] += w22;
        // H_rr = -[q]x W (upper): rows of -[q]x are (0, qz, -qy), (-qz, 0, qx), (qy, -qx, 0)
        acc[15] += fqz * w10 - fqy * w20;
        acc[16] += fqz * w11 - fqy * w21;
        acc[17] += fqz * w12 - fqy * w22;
        acc[18] += fqx * w21 - fqz * w01;
        acc[19] += fqx * w22 - fqz * w02;
        acc[20] += fqy * w02 - fqx * w12;
      }
    }
  }

  // ---- tile reduction: fp64 warp shuffles, then fixed-order across warps
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int j = 0; j < kNumTerms; ++j) {
    double s = warp_sum((double)acc[j]);
    if (lane == 0) red[warp][j] = s;
  }
#pragma unroll
  for (int l = 0; l < GVOX_MAX_LEVELS; ++l) {
    int s = l < MAXL ? warp_sum_i(inl[l < MAXL ? l : 0]) : 0;
    if (lane == 0) red[warp][28 + l] = (double)s;
  }
  {
    int s1 = warp_sum_i(n_invisible), s2 = warp_sum_i(n_degenerate);
    if (lane == 0) {
      red[warp][36] = (double)s1;
      red[warp][37] = (double)s2;
      red[warp][38] = 0.0;
      red[warp][39] = 0.0;
    }
  }
  __syncthreads();
  if (tid < kPartialStride) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += red[w][tid];
    partials[tile * kPartialStride + tid] = s;
  }
}

// ---------------------------------------------------------------- K4 / expand

// Ad(T) for rotation-first tangents: [[R, 0], [t^ R, R]] (row-major 6x6).
__device__ inline void adjoint6(const double* R, const double* t, double* Ad) {
  for (int i = 0; i < 36; ++i) Ad[i] = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      Ad[a * 6 + b] = R[a * 3 + b];
      Ad[(a + 3) * 6 + (b + 3)] = R[a * 3 + b];
    }
  // [t]x R
  const double T[9] = {0, -t[2], t[1], t[2], 0, -t[0], -t[1], t[0], 0};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double s = 0;
      for (int c = 0; c < 3; ++c) s += T[a * 3 + c] * R[c * 3 + b];
      Ad[(a + 3) * 6 + b] = s;
    }
}

// compact terms (upper H_jj 21, b_j 6, e) -> full record.  One warp per record.
__device__ void expand_warp(const double* terms, const int32_t* counts, const double* Ti,
                            const double* Tj, gvox_linear_factor* out, double* scratch) {
  // scratch: [36 H] [36 Ad] [36 M=H Ad] [6 b]
  const int lane = threadIdx.x & 31;
  double* H = scratch;
  double* Ad = scratch + 36;
  double* M = scratch + 72;
  if (lane == 0) {
    double R[9], t[3], v[3];
    relative_pose_dev(Ti, Tj, R, t, v);
    adjoint6(R, t, Ad);
    int k = 0;
    for (int r = 0; r < 6; ++r)
      for (int c = r; c < 6; ++c) {
        H[r * 6 + c] = terms[k];
        H[c * 6 + r] = terms[k];
        ++k;
      }
  }
  __syncwarp();
  for (int e = lane; e < 36; e += 32) {
    int r = e / 6, c = e % 6;
    double s = 0;
    for (int k = 0; k < 6; ++k) s += H[r * 6 + k] * Ad[k * 6 + c];
    M[e] = s;
  }
  __syncwarp();
  for (int e = lane; e < 36; e += 32) {
    int r = e / 6, c = e % 6;
    double sii = 0, sij = 0;
    for (int k = 0; k < 6; ++k) {
      sii += Ad[k * 6 + r] * M[k * 6 + c];
      sij += Ad[k * 6 + r] * H[k * 6 + c];
    }
    out->H_ii[e] = sii;
    out->H_ij[e] = -sij;
    out->H_jj[e] = H[e];
  }
  if (lane < 6) {
    double s = 0;
    for (int k = 0; k < 6; ++k) s += Ad[k * 6 + lane] * terms[21 + k];
    out->b_i[lane] = -s;
    out->b_j[lane] = terms[21 + lane];
  }
  if (lane < GVOX_MAX_LEVELS) out->inliers[lane] = counts[lane];
  if (lane == 0) {
    out->error = terms[27];
    out->num_invisible = counts[8];
    out->num_degenerate = counts[9];
  }
}

// internal tile-term order -> compact (upper triangle of H_jj, b_j, e)
__device__ inline void internal_to_compact(const double* t, double* c) {
  // H_jj = [[H_rr, H_rt], [H_tr, H_tt]], H_rt = -W^T, H_tt = Omega
  const double Hrr[9] = {t[15], t[16], t[17], t[16], t[18], t[19], t[17], t[19], t[20]};
  const double* W = t + 6;
  const double Om[9] = {t[0], t[1], t[2], t[1], t[3], t[4], t[2], t[4], t[5]};
  double H[36];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      H[a * 6 + b] = Hrr[a * 3 + b];
      H[a * 6 + 3 + b] = -W[b * 3 + a];
      H[(a + 3) * 6 + b] = -W[a * 3 + b];
      H[(a + 3) * 6 + 3 + b] = Om[a * 3 + b];
    }
  int k = 0;
  for (int r = 0; r < 6; ++r)
    for (int cc = r; cc < 6; ++cc) c[k++] = H[r * 6 + cc];
  for (int j = 0; j < 3; ++j) {
    c[21 + j] = t[21 + j];
    c[24 + j] = t[24 + j];
  }
  c[27] = t[27];
}

constexpr int kReduceWarps = 4;

__global__ void k_reduce(const FactorDev* __restrict__ factors, const int32_t* __restrict__ tile_start,
                         int64_t num_factors, const double* __restrict__ poses,
                         const double* __restrict__ partials, gvox_linear_factor* __restrict__ out_full,
                         gvox_factor_accum* __restrict__ out_accum) {
  __shared__ double sum_s[kReduceWarps][kPartialStride];
  __shared__ double comp_s[kReduceWarps][28];
  __shared__ int32_t cnt_s[kReduceWarps][10];
  __shared__ double scratch_s[kReduceWarps][108];
  __shared__ double pose_s[kReduceWarps][24];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t f = (int64_t)blockIdx.x * kReduceWarps + w;
  if (f >= num_factors) return;
  const int32_t t0 = tile_start[f], t1 = tile_start[f + 1];
  // fixed tile order -> deterministic sums
  for (int j = lane; j < kPartialStride; j += 32) {
    double s = 0.0;
    for (int32_t t = t0; t < t1; ++t) s += partials[(int64_t)t * kPartialStride + j];
    sum_s[w][j] = s;
  }
  __syncwarp();
  if (lane == 0) {
    internal_to_compact(sum_s[w], comp_s[w]);
    for (int l = 0; l < 8; ++l) cnt_s[w][l] = (int32_t)sum_s[w][28 + l];
    cnt_s[w][8] = (int32_t)sum_s[w][36];
    cnt_s[w][9] = (int32_t)sum_s[w][37];
  }
  __syncwarp();
  if (out_accum) {
    gvox_factor_accum* o = out_accum + f;
    if (lane < 28) o->terms[lane] = comp_s[w][lane];
    if (lane < 8) o->inliers[lane] = cnt_s[w][lane];
    if (lane == 0) {
      o->num_invisible = cnt_s[w][8];
      o->num_degenerate = cnt_s[w][9];
    }
    if (lane < 6) o->reserved[lane] = 0;
    return;
  }
  const FactorDev fd = factors[f];
  if (lane < 24) pose_s[w][lane] = poses[12 * (int64_t)(lane < 12 ? fd.pi : fd.pj) + (lane % 12)];
  __syncwarp();
  expand_warp(comp_s[w], cnt_s[w], pose_s[w], pose_s[w] + 12, out_full + f, scratch_s[w]);
}

__global__ void k_expand(const FactorDev* __restrict__ factors, int64_t num_factors,
                         const double* __restrict__ poses, const gvox_factor_accum* __restrict__ accum,
                         gvox_linear_factor* __restrict__ out) {
  __shared__ double comp_s[kReduceWarps][28];
  __shared__ int32_t cnt_s[kReduceWarps][10];
  __shared__ double scratch_s[kReduceWarps][108];
  __shared__ double pose_s[kReduceWarps][24];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t f = (int64_t)blockIdx.x * kReduceWarps + w;
  if (f >= num_factors) return;
  const gvox_factor_accum* a = accum + f;
  if (lane < 28) comp_s[w][lane] = a->terms[lane];
  if (lane < 8) cnt_s[w][lane] = a->inliers[lane];
  if (lane == 0) {
    cnt_s[w][8] = a->num_invisible;
    cnt_s[w][9] = a->num_degenerate;
  }
  const FactorDev fd = factors[f];
  if (lane < 24) pose_s[w][lane] = poses[12 * (int64_t)(lane < 12 ? fd.pi : fd.pj) + (lane % 12)];
  __syncwarp();
  expand_warp(comp_s[w], cnt_s[w], pose_s[w], pose_s[w] + 12, out + f, scratch_s[w]);
}

}  // namespace

void launch_linearize(const CloudDev* const* clouds, const MapDev* const* maps,
                      const FactorDev* factors, const int32_t* tile_start, int64_t num_factors,
                      int64_t num_tiles, int tile_pts, int max_levels, const double* poses,
                      double* partials, int32_t* tile_factor, int64_t* corr_dump,
                      bool all_dense, cudaStream_t stream) {
  if (num_tiles <= 0) return;
  const unsigned grid = (unsigned)num_tiles;
  if (max_levels <= 3) {
    if (all_dense)
      k_linearize<3, true><<<grid, kThreads, 0, stream>>>(clouds, maps, factors, tile_start,
                                                          tile_factor, tile_pts, poses, partials,
                                                          corr_dump);
    else
      k_linearize<3, false><<<grid, kThreads, 0, stream>>>(clouds, maps, factors, tile_start,
                                                           tile_factor, tile_pts, poses, partials,
                                                           corr_dump);
  } else {
    k_linearize<GVOX_MAX_LEVELS, false><<<grid, kThreads, 0, stream>>>(
        clouds, maps, factors, tile_start, tile_factor, tile_pts, poses, partials, corr_dump);
  }
  note_launch();
}

void launch_tile_map(const int32_t* tile_start, int64_t num_items, int32_t* tile_owner,
                     cudaStream_t stream) {
  if (num_items <= 0) return;
  k_tile_map<<<(unsigned)((num_items + 255) / 256), 256, 0, stream>>>(tile_start, num_items,
                                                                      tile_owner);
  note_launch();
}

void launch_reduce(const FactorDev* factors, const int32_t* tile_start, int64_t num_factors,
                   const double* poses, const double* partials, gvox_linear_factor* out_full,
                   gvox_factor_accum* out_accum, cudaStream_t stream) {
  if (num_factors <= 0) return;
  unsigned blocks = (unsigned)((num_factors + kReduceWarps - 1) / kReduceWarps);
  k_reduce<<<blocks, 32 * kReduceWarps, 0, stream>>>(factors, tile_start, num_factors, poses,
                                                     partials, out_full, out_accum);
  note_launch();
}

void launch_expand(const FactorDev* factors, int64_t num_factors, const double* poses,
                   const gvox_factor_accum* accum, gvox_linear_factor* out, cudaStream_t stream) {
  if (num_factors <= 0) return;
  unsigned blocks = (unsigned)((num_factors + kReduceWarps - 1) / kReduceWarps);
  k_expand<<<blocks, 32 * kReduceWarps, 0, stream>>>(factors, num_factors, poses, accum, out);
  note_launch();
}

}  // namespace gvox
