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

// Tuning knobs (compile-time; defaults are the measured best on B200, see
// tools/variants.py).  Measured on C5 (r01): 128 x 4 CTAs/SM 197 ms, 256 x 2
// 204 ms; forcing 3 CTAs of 256 (80 registers) spills, 280 ms; one level at a
// time (G = 1) 264 ms; a cp.async two-stage pipeline through shared memory
// (records + point data, 224 B per point slot) 328 ms at 12 warps/SM.
#ifndef GVOX_LIN_THREADS
#define GVOX_LIN_THREADS 128
#endif
#ifndef GVOX_LIN_MINB
#define GVOX_LIN_MINB 4
#endif
#ifndef GVOX_LIN_G
#define GVOX_LIN_G 4
#endif
// source prefetch: 0 = per-thread cp.async (LDGSTS), 1 = per-warp bulk copy + mbarrier
#ifndef GVOX_LIN_BULK
#define GVOX_LIN_BULK 0
#endif
#ifndef GVOX_LIN_PIPE
#define GVOX_LIN_PIPE 1
#endif
// exact chunk culling against the coarsest level's occupancy (FAST pipeline)
#ifndef GVOX_LIN_CULL
#define GVOX_LIN_CULL 1
#endif
#ifndef GVOX_LIN_STAGES
#define GVOX_LIN_STAGES (GVOX_LIN_PIPE ? 3 : 2)
#endif
// FAST all-dense probes: one bounds test per point on the nested grid boxes (1)
// or one per level (0; both correct on nested boxes)
#ifndef GVOX_LIN_NESTED
#define GVOX_LIN_NESTED 1
#endif
// residual base of level l > 0 from level l - 1's (one select + add per axis, 1)
// or from the level-0 base and the key's low bits (0)
#ifndef GVOX_LIN_INCBASE
#define GVOX_LIN_INCBASE 1
#endif
// level term: 1/det folded into the level sums' FMAs and into g (1), or Omega
// formed explicitly first (0)
#ifndef GVOX_LIN_FUSEOM
#define GVOX_LIN_FUSEOM 1
#endif
// FAST pipeline: loop unrolled twice with the current / next point's data in
// alternating register sets (1), or one set copied into the other (0)
#ifndef GVOX_LIN_UNROLL2
#define GVOX_LIN_UNROLL2 1
#endif
// FAST all-dense pipeline three points deep with the voxel records gathered
// into shared memory by cp.async one point ahead (1), or the two-point register
// pipeline (0); GVOX_LIN_DEEP_CG: the 16-byte record gathers bypass L1 (1).
// Measured (r02aa, full C5, ncu): DEEP 248.6 ms vs 121.9 -- 17 % more
// instructions (LDGSTS + LDS per record word), short_scoreboard 4.1 and
// mio_throttle 1.1 cycles/issue, and the grid probes now wait (44 KB of shared
// memory per CTA leaves L1 a third of its size): rejected, kept for the record.
#ifndef GVOX_LIN_DEEP
#define GVOX_LIN_DEEP 0
#endif
#ifndef GVOX_LIN_DEEP_CG
#define GVOX_LIN_DEEP_CG 0
#endif
// FAST all-dense pipeline three points deep in REGISTERS (1): the grid probes
// two points ahead, the voxel records gathered one point ahead into registers
// (a 4-stage source ring); needs more registers per thread (build with
// GVOX_LIN_MINB=3)
#ifndef GVOX_LIN_RPIPE
#define GVOX_LIN_RPIPE 0
#endif
// FAST two-point pipeline, order inside a live iteration: 0 = prep of the next
// point, gathers, R C R^T, level terms; 1 = prep, R C R^T, gathers, level terms
// (ncu: the first R C R^T instruction after the gathers waited on their
// scoreboard); 2 = gathers, then prep of the next point, R C R^T, level terms
#ifndef GVOX_LIN_ORDER
#define GVOX_LIN_ORDER 0
#endif
// culling pass: the next pass's chunk boxes prefetched (1)
#ifndef GVOX_CULL_PREFETCH
#define GVOX_CULL_PREFETCH 1
#endif


constexpr int kThreads = GVOX_LIN_THREADS;
constexpr int kWarps = kThreads / 32;

struct FactorShared {
  double R[9];
  double t[3];
  double v[3];
  float Rf[9];
  // the rotation's columns 0-2, rows 0 and 1, as packed pairs (R0, R3), (R1, R4),
  // (R2, R5): one 8-byte shared load lands a pair in an aligned register pair,
  // ready for the packed FMAs of R C R^T (no register moves to form them)
  f2_t Rp[3];
  const float4* A;  // the tile's chunked point records (B = A + 32, N = A + 64 per chunk)
  const float* cbox;  // the tile's first chunk box (6 floats per chunk)
  int64_t begin, end;
  int64_t corr_base;
  double r0, inv_r0;
  int L, dyadic, validate, error_only;
  MapLevelDev lv[GVOX_MAX_LEVELS];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16_s(unsigned s, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
// L1-allocating copies (the record gathers: neighbouring points share voxels)
__device__ __forceinline__ void cp_async16_ca(unsigned s, const void* gmem) {
#if GVOX_LIN_DEEP_CG
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
#else
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
#endif
}
__device__ __forceinline__ void cp_async4_ca(unsigned s, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// all but the newest N groups have landed
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// mbarrier + bulk copy (async proxy) helpers
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// Dense-grid probe without branches: the load is predicated on the bounds test.
__device__ __forceinline__ int32_t lookup_dense_pred(const MapLevelDev& lv, int32_t kx, int32_t ky,
                                                     int32_t kz) {
  const int4 b0 = *reinterpret_cast<const int4*>(&lv.x0);   // x0 y0 z0 dx
  const uint4 b1 = *reinterpret_cast<const uint4*>(&lv.dy);  // dy dz syz dense
  const uint32_t cx = (uint32_t)(kx - b0.x), cy = (uint32_t)(ky - b0.y), cz = (uint32_t)(kz - b0.z);
  const bool in = (cx < (uint32_t)b0.w) & (cy < b1.x) & (cz < b1.y);
  int32_t v = -1;
  if (in) v = __ldg(lv.grid + (cx * b1.z + cy * b1.y + cz));
  return v;
}

// All-dense maps of this library have NESTED grid boxes (gvox_runtime.cu build
// plan: level l's box is the coarsest box refined, x0_l = x0_0 >> l, d_l =
// d_0 >> l), so the level-0 bounds test decides every level and the level-l
// cell is the level-0 cell offset shifted: one subtraction and one unsigned
// compare per axis per POINT instead of per level.
template <int MAXL>
__device__ __forceinline__ void lookup_nested(const MapLevelDev* lv, int32_t kx, int32_t ky,
                                              int32_t kz, int32_t* vid) {
  const int4 b0 = *reinterpret_cast<const int4*>(&lv[0].x0);  // x0 y0 z0 dx
  const uint4 b1 = *reinterpret_cast<const uint4*>(&lv[0].dy);  // dy dz syz dense
  const uint32_t cx = (uint32_t)(kx - b0.x), cy = (uint32_t)(ky - b0.y), cz = (uint32_t)(kz - b0.z);
  const bool in = (cx < (uint32_t)b0.w) & (cy < b1.x) & (cz < b1.y);
#pragma unroll
  for (int l = 0; l < MAXL; ++l) {
    const uint4 bl = l == 0 ? b1 : *reinterpret_cast<const uint4*>(&lv[l].dy);
    int32_t v = -1;
    if (in) v = __ldg(lv[l].grid + ((cx >> l) * bl.z + (cy >> l) * bl.y + (cz >> l)));
    vid[l] = v;
  }
}

// 1/x for x > 0 finite (MUFU.RCP, ~1 ulp)
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__global__ void k_tile_map(const int32_t* __restrict__ tile_start, int64_t num_factors,
                           int32_t* __restrict__ tile_factor) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= num_factors) return;
  for (int32_t t = tile_start[f]; t < tile_start[f + 1]; ++t) tile_factor[t] = (int32_t)f;
}

// ---------------------------------------------------------------- shared parts

// Per-thread fp32 accumulators (packed pairs where the algebra pairs up).
template <int MAXL>
struct Acc {
  f2_t A = 0, C = 0;            // sum (o00, o01), sum (o02, o12)
  float o11 = 0.f, o22 = 0.f;
  f2_t W0 = 0, W1 = 0, W2 = 0;  // sum (W0j, W1j), j = 0, 1, 2  (W = Omega [q]x)
  float W20 = 0.f, W21 = 0.f, W22 = 0.f;
  float h00 = 0.f, h01 = 0.f, h02 = 0.f, h11 = 0.f, h12 = 0.f, h22 = 0.f;  // sum -[q]x W
  f2_t X = 0, Y = 0;  // sum qz (gx, gy), sum gz (qy, qx)  -> b_rot xy
  float rz = 0.f;     // sum (q x g)_z
  f2_t G = 0;         // sum (gx, gy)
  float gz = 0.f;
  f2_t E = 0;         // sum (dx gx, dy gy)
  float ez = 0.f;
  int inl[MAXL];
  int n_invisible = 0, n_degenerate = 0;
  __device__ Acc() {
#pragma unroll
    for (int l = 0; l < MAXL; ++l) inl[l] = 0;
  }
};

// Per-point quantities shared by its levels.
struct PointData {
  float qx, qy, qz;   // T_ij mu (fp32 lever arm)
  float ex, ey, ez;   // centre_0 - q (level-0 residual base)
  f2_t Sp1, Sp2;      // (s01, s11), (s02, s12) of R C R^T
  float s00, s22;
  int32_t k0x, k0y, k0z;  // level-0 key (the grid probes)
  uint32_t kb;            // low 8 bits of k0x | k0y << 8 | k0z << 16 (level residual bases)
};

// Stage the factor of `tile` in shared memory (pose, cloud, map levels).
template <int MAXL>
__device__ __forceinline__ void stage_factor(FactorShared& sh, double* pose_s,
                                             const CloudDev* const* clouds, const MapDev* const* maps,
                                             const FactorDev* factors, const int32_t* tile_start,
                                             const int32_t* tile_factor, int tile_pts,
                                             const double* poses, int64_t tile) {
  const int tid = threadIdx.x;
  const int32_t f = __ldg(tile_factor + tile);
  const FactorDev fd = factors[f];
  if (tid < 24) {
    pose_s[tid] = __ldg(poses + 12 * (int64_t)(tid < 12 ? fd.pi : fd.pj) + (tid % 12));
  } else if (tid == 32) {
    const CloudDev* cd = clouds[fd.src];
    int64_t b = (int64_t)(tile - __ldg(tile_start + f)) * fd.tile_pts;
    int64_t e = b + fd.tile_pts;
    int64_t n = cd->n;
    sh.A = cd->A + pt_off(b);  // the tile's first chunk (tiles are chunk-aligned)
    sh.cbox = cd->chunk_box ? cd->chunk_box + 6 * (b >> 5) : nullptr;
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
#pragma unroll
    for (int j = 0; j < 3; ++j) sh.Rp[j] = pk(sh.Rf[j], sh.Rf[3 + j]);
  }
  __syncthreads();
}

// P:197 visibility test: true if the point is discarded.
__device__ __forceinline__ bool invisible(const FactorShared& sh, const float4 a, const float4 c) {
  if (c.y == 0.f && c.z == 0.f && c.w == 0.f) return false;  // zero normal: no test (Q7)
  const double dx = (double)a.x - sh.v[0], dy = (double)a.y - sh.v[1], dz = (double)a.z - sh.v[2];
  const double dot = __fma_rn(dx, (double)c.y, __fma_rn(dy, (double)c.z, __dmul_rn(dz, (double)c.w)));
  return dot > 0.0;
}

// q = T_ij mu (fp64, pinned order, Q10), level-0 key, fp32 residual base.
__device__ __forceinline__ void transform_point(const FactorShared& sh, const float4 a, int dyadic,
                                                double r0, double inv_r0, float r0f, PointData& pd) {
  const double mx = a.x, my = a.y, mz = a.z;
  const double qx = __fma_rn(sh.R[0], mx, __fma_rn(sh.R[1], my, __fma_rn(sh.R[2], mz, sh.t[0])));
  const double qy = __fma_rn(sh.R[3], mx, __fma_rn(sh.R[4], my, __fma_rn(sh.R[5], mz, sh.t[1])));
  const double qz = __fma_rn(sh.R[6], mx, __fma_rn(sh.R[7], my, __fma_rn(sh.R[8], mz, sh.t[2])));
  // saturating floor: a saturated coordinate misses every grid / fails key_in_range
  pd.k0x = voxel_coord0(qx, r0, inv_r0, dyadic);
  pd.k0y = voxel_coord0(qy, r0, inv_r0, dyadic);
  pd.k0z = voxel_coord0(qz, r0, inv_r0, dyadic);
  pd.qx = (float)qx;
  pd.qy = (float)qy;
  pd.qz = (float)qz;
  pd.kb = ((uint32_t)pd.k0x & 0xffu) | (((uint32_t)pd.k0y & 0xffu) << 8) |
          (((uint32_t)pd.k0z & 0xffu) << 16);
  pd.ex = 0.5f * r0f - (float)(qx - (double)pd.k0x * r0);
  pd.ey = 0.5f * r0f - (float)(qy - (double)pd.k0y * r0);
  pd.ez = 0.5f * r0f - (float)(qz - (double)pd.k0z * r0);
}

// R C R^T (symmetric) in packed pairs over rows 0/1: M = R C by columns, S = M R^T.
__device__ __forceinline__ void rcr(const float* R, const f2_t* Rp, const float4 a, const float4 b,
                                    const float4 c, PointData& pd) {
  const float c00 = a.w, c01 = b.x, c02 = b.y, c11 = b.z, c12 = b.w, c22 = c.x;
  const f2_t Rc0 = Rp[0], Rc1 = Rp[1], Rc2 = Rp[2];  // (R0, R3), (R1, R4), (R2, R5)
  const f2_t Mp0 = fma2(Rc2, bc(c02), fma2(Rc1, bc(c01), mul2(Rc0, bc(c00))));
  const f2_t Mp1 = fma2(Rc2, bc(c12), fma2(Rc1, bc(c11), mul2(Rc0, bc(c01))));
  const f2_t Mp2 = fma2(Rc2, bc(c22), fma2(Rc1, bc(c12), mul2(Rc0, bc(c02))));
  const float M20 = fmaf(R[8], c02, fmaf(R[7], c01, R[6] * c00));
  const float M21 = fmaf(R[8], c12, fmaf(R[7], c11, R[6] * c01));
  const float M22 = fmaf(R[8], c22, fmaf(R[7], c12, R[6] * c02));
  const f2_t Sp0 = fma2(Mp2, bc(R[2]), fma2(Mp1, bc(R[1]), mul2(Mp0, bc(R[0]))));  // (s00, s10)
  pd.Sp1 = fma2(Mp2, bc(R[5]), fma2(Mp1, bc(R[4]), mul2(Mp0, bc(R[3]))));          // (s01, s11)
  pd.Sp2 = fma2(Mp2, bc(R[8]), fma2(Mp1, bc(R[7]), mul2(Mp0, bc(R[6]))));          // (s02, s12)
  pd.s00 = lo(Sp0);
  pd.s22 = fmaf(M22, R[8], fmaf(M21, R[7], M20 * R[6]));
}

// Level folding.  B_k = [-(q)x, I] depends on the point only, so for one point
//   sum_l B^T Omega_l B = B^T (sum_l Omega_l) B,   sum_l B^T Omega_l d_l = B^T (sum_l g_l)
// with g_l = Omega_l d_l.  Each hit level therefore only adds its Omega_l and
// g_l into per-point sums (level_term); the q-dependent target-block terms are
// accumulated once per point (fold_point).  Exact algebra; only the fp32
// summation order changes.
struct LevelSum {
  f2_t Oa, Oc;   // sum (o00, o01), sum (o02, o12)
  float o11, o22;
  f2_t G;        // sum (gx, gy)
  float gz;
};

// Residual base of level l, centre_l - q, in fp32 (reading Q12: the fp64 part
// is the level-0 base pd.e = centre_0 - q).  Call for l = 0, 1, ... in order
// with (bx, by, bz) = pd.e before level 0.
//  INCBASE 0: with k_l = k0 >> l, centre_l - q = (centre_0 - q)
//             + r0 (2^(l-1) - 1/2 - (k0 & (2^l - 1)))   (from level 0 each time)
//  INCBASE 1: centre_l - centre_(l-1) = r_(l-1) (1/2 - bit_(l-1)(k0)), so each
//             level adds +-r_(l-1)/2 to the previous level's base
__device__ __forceinline__ void level_base(const PointData& pd, const int l, const float r0f,
                                           float& bx, float& by, float& bz) {
  if (l == 0) return;
#if GVOX_LIN_INCBASE
  const float h = 0.5f * r0f * (float)(1 << (l - 1));  // exact: a power-of-two multiple
  bx += ((pd.kb >> (l - 1)) & 1u) ? -h : h;
  by += ((pd.kb >> (l + 7)) & 1u) ? -h : h;
  bz += ((pd.kb >> (l + 15)) & 1u) ? -h : h;
#else
  const int mlo = (1 << l) - 1;
  const float sh_l = 0.5f * (float)(1 << l) - 0.5f;
  bx = fmaf(r0f, sh_l - (float)(pd.kb & mlo), pd.ex);
  by = fmaf(r0f, sh_l - (float)((pd.kb >> 8) & mlo), pd.ey);
  bz = fmaf(r0f, sh_l - (float)((pd.kb >> 16) & mlo), pd.ez);
#endif
}

// One (point, level) term: Eq.3 fused covariance, Omega, residual, g = Omega d,
// e = d^T g.  v0 = {off.xyz, C.xx}, v1 = {C.xy, C.yy, C.xz, C.yz}, v2 = C.zz.
template <int MAXL>
__device__ __forceinline__ void level_term(Acc<MAXL>& ac, LevelSum& ls, const PointData& pd,
                                           const float4 v0, const float4 v1, const float v2,
                                           const int l, const float bx, const float by,
                                           const float bz, const bool hit = true) {
  // fused covariance (Eq.3)
  const f2_t P = add2(pk(v1.x, v1.y), pd.Sp1);  // (cb, cd) = (xy, yy)
  const f2_t Q = add2(pk(v1.z, v1.w), pd.Sp2);  // (cc, ce) = (xz, yz)
  const float ca = v0.w + pd.s00, cf = v2 + pd.s22;
  const float cb = lo(P), cd = hi(P), cc = lo(Q), ce = hi(Q);
  // inverse by the symmetric adjugate
  const float i00 = fmaf(cd, cf, -ce * ce);
  const float i01 = fmaf(cc, ce, -cb * cf);
  const float i02 = fmaf(cb, ce, -cc * cd);
  const float i11 = fmaf(ca, cf, -cc * cc);
  const float i12 = fmaf(cb, cc, -ca * ce);
  const float i22 = fmaf(ca, cd, -cb * cb);
  const float det = fmaf(ca, i00, fmaf(cb, i01, cc * i02));
  // Q16: a fused covariance that is not positive definite contributes nothing
  // det >= FLT_MIN (normal) and finite  <=>  bits(det) - bits(FLT_MIN) <
  // bits(FLT_MAX) - bits(FLT_MIN) + 1 (unsigned): a subnormal det would make the
  // flush-to-zero reciprocal +Inf and poison the factor (reading R22)
  const bool pd_ok = __float_as_uint(det) - 0x00800000u < 0x7F7FFFFFu - 0x007FFFFFu;
  // (hit = false: a level without a correspondence, evaluated branch-free and
  // masked out -- Omega = 0 makes every contribution below exactly zero)
  const bool ok = pd_ok && hit;
  const float id = ok ? rcp_approx(det) : 0.f;
  ac.n_degenerate += hit && !pd_ok;
  ac.inl[l] += ok;
#if GVOX_LIN_FUSEOM
  // d = mu~ - q = (centre_l - q) + offset (Q12); (bx, by, bz) = centre_l - q
  // from level_base
  const f2_t D = add2(pk(bx, by), pk(v0.x, v0.y));  // (dx, dy)
  const float dz = bz + v0.z;
  const float dx = lo(D), dy = hi(D);
  // g = Omega d = (adj d) / det, e = d^T g; Omega = adj / det enters the level
  // sums through one FMA per pair
  const f2_t A01 = pk(i00, i01), A11 = pk(i01, i11), A12 = pk(i02, i12);
  const f2_t Tp = fma2(A12, bc(dz), fma2(A11, bc(dy), mul2(A01, bc(dx))));
  const float tz = fmaf(i02, dx, fmaf(i12, dy, i22 * dz));
  const f2_t Gp = mul2(Tp, bc(id));  // (gx, gy)
  const float gz = tz * id;
  ac.E = fma2(D, Gp, ac.E);
  ac.ez = fmaf(dz, gz, ac.ez);
  ls.Oa = fma2(A01, bc(id), ls.Oa);
  ls.Oc = fma2(A12, bc(id), ls.Oc);
  ls.o11 = fmaf(i11, id, ls.o11);
  ls.o22 = fmaf(i22, id, ls.o22);
  ls.G = add2(ls.G, Gp);
  ls.gz += gz;
#else
  const f2_t Om_a = mul2(pk(i00, i01), bc(id));  // (o00, o01) = column 0, rows 0-1
  const f2_t Om_b = mul2(pk(i01, i11), bc(id));  // (o01, o11) = column 1, rows 0-1
  const f2_t Om_c = mul2(pk(i02, i12), bc(id));  // (o02, o12) = column 2, rows 0-1
  const float o22 = i22 * id;

  // d = mu~ - q = (centre_l - q) + offset (Q12); (bx, by, bz) = centre_l - q
  // from level_base
  const f2_t D = add2(pk(bx, by), pk(v0.x, v0.y));  // (dx, dy)
  const float dz = bz + v0.z;
  const float dx = lo(D), dy = hi(D);

  // g = Omega d, e = d^T g
  const f2_t Gp = fma2(Om_c, bc(dz), fma2(Om_b, bc(dy), mul2(Om_a, bc(dx))));  // (gx, gy)
  const float gz = fmaf(lo(Om_c), dx, fmaf(hi(Om_c), dy, o22 * dz));
  ac.E = fma2(D, Gp, ac.E);
  ac.ez = fmaf(dz, gz, ac.ez);
  // per-point level sums
  ls.Oa = add2(ls.Oa, Om_a);
  ls.Oc = add2(ls.Oc, Om_c);
  ls.o11 += hi(Om_b);
  ls.o22 += o22;
  ls.G = add2(ls.G, Gp);
  ls.gz += gz;
#endif
}

// The target-block terms of one point from its level sums (Eqs.6-8 with
// B = [-(q)x, I]): sum Omega, W = Omega [q]x, -[q]x W, q x g, g.
template <int MAXL>
__device__ __forceinline__ void fold_point(Acc<MAXL>& ac, const LevelSum& ls, const PointData& pd) {
  const float qx = pd.qx, qy = pd.qy, qz = pd.qz;
  const f2_t Om_a = ls.Oa, Om_c = ls.Oc;                  // (o00, o01), (o02, o12)
  const f2_t Om_b = pk(hi(ls.Oa), ls.o11);                  // (o01, o11)
  const float o22 = ls.o22, o02 = lo(Om_c), o12 = hi(Om_c);
  const f2_t Gp = ls.G;
  const float gz = ls.gz, gx = lo(Gp), gy = hi(Gp);
  ac.G = add2(ac.G, Gp);
  ac.gz += gz;
  // b_rot = q x g, with X = sum qz (gx, gy), Y = sum gz (qy, qx):
  // brx = Y.x - X.y, bry = X.x - Y.y (combined at the tile reduction)
  ac.X = fma2(bc(qz), Gp, ac.X);
  ac.Y = fma2(bc(gz), pk(qy, qx), ac.Y);
  ac.rz = fmaf(qx, gy, fmaf(-qy, gx, ac.rz));
  // sum Omega
  ac.A = add2(ac.A, Om_a);
  ac.C = add2(ac.C, Om_c);
  ac.o11 += ls.o11;
  ac.o22 += o22;
  // W = Omega [q]x by columns: W[:,0] = qz Om[:,1] - qy Om[:,2],
  // W[:,1] = qx Om[:,2] - qz Om[:,0], W[:,2] = qy Om[:,0] - qx Om[:,1]
  const f2_t Wc0 = fma2(bc(-qy), Om_c, mul2(bc(qz), Om_b));
  const f2_t Wc1 = fma2(bc(qx), Om_c, mul2(bc(-qz), Om_a));
  const f2_t Wc2 = fma2(bc(-qx), Om_b, mul2(bc(qy), Om_a));
  const float W20 = fmaf(qz, o12, -qy * o22);
  const float W21 = fmaf(qx, o22, -qz * o02);
  const float W22 = fmaf(qy, o02, -qx * o12);
  ac.W0 = add2(ac.W0, Wc0);
  ac.W1 = add2(ac.W1, Wc1);
  ac.W2 = add2(ac.W2, Wc2);
  ac.W20 += W20;
  ac.W21 += W21;
  ac.W22 += W22;
  // H_rr = -[q]x W (upper)
  ac.h00 = fmaf(qz, hi(Wc0), fmaf(-qy, W20, ac.h00));
  ac.h01 = fmaf(qz, hi(Wc1), fmaf(-qy, W21, ac.h01));
  ac.h02 = fmaf(qz, hi(Wc2), fmaf(-qy, W22, ac.h02));
  ac.h11 = fmaf(qx, W21, fmaf(-qz, lo(Wc1), ac.h11));
  ac.h12 = fmaf(qx, W22, fmaf(-qz, lo(Wc2), ac.h12));
  ac.h22 = fmaf(qy, lo(Wc2), fmaf(-qx, hi(Wc2), ac.h22));
}

// Tile reduction: fp64 warp shuffles, then a fixed-order sum across warps.
// Internal term order t[0..27] (see the file header).
template <int MAXL>
__device__ __forceinline__ void tile_reduce(const Acc<MAXL>& ac, double (*red)[kPartialStride],
                                            double* partials, int64_t tile) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  {
    const double t[27] = {lo(ac.A), hi(ac.A), lo(ac.C), ac.o11, hi(ac.C), ac.o22,
                          lo(ac.W0), lo(ac.W1), lo(ac.W2), hi(ac.W0), hi(ac.W1), hi(ac.W2),
                          ac.W20, ac.W21, ac.W22,
                          ac.h00, ac.h01, ac.h02, ac.h11, ac.h12, ac.h22,
                          (double)lo(ac.Y) - (double)hi(ac.X), (double)lo(ac.X) - (double)hi(ac.Y),
                          ac.rz, lo(ac.G), hi(ac.G), ac.gz};
#pragma unroll
    for (int j = 0; j < 27; ++j) {
      double s = warp_sum(t[j]);
      if (lane == 0) red[warp][j] = s;
    }
    double e = warp_sum((double)lo(ac.E) + (double)hi(ac.E) + (double)ac.ez);
    if (lane == 0) red[warp][27] = e;
  }
#pragma unroll
  for (int l = 0; l < GVOX_MAX_LEVELS; ++l) {
    int s = l < MAXL ? warp_sum_i(ac.inl[l < MAXL ? l : 0]) : 0;
    if (lane == 0) red[warp][28 + l] = (double)s;
  }
  {
    int s1 = warp_sum_i(ac.n_invisible), s2 = warp_sum_i(ac.n_degenerate);
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

// ---------------------------------------------------------------- K3
// Source records are prefetched S - 1 iterations ahead into a per-warp ring in
// shared memory: per-thread cp.async (LDGSTS, default) or, with GVOX_LIN_BULK,
// one lane per warp arming an mbarrier and issuing three cp.async.bulk copies
// (the A, B, N planes of the warp's next 32 points).  FAST is the specialisation for the common
// batch (exactly MAXL dyadic levels, no visibility test, no correspondence
// dump): no runtime level / flag tests and branch-free grid probes.
template <int MAXL, bool ALL_DENSE, bool FAST, bool VALID = false>
__global__ void __launch_bounds__(kThreads, GVOX_LIN_MINB)
    k_linearize(const CloudDev* const* __restrict__ clouds, const MapDev* const* __restrict__ maps,
                const FactorDev* __restrict__ factors, const int32_t* __restrict__ tile_start,
                const int32_t* __restrict__ tile_factor, int tile_pts,
                const double* __restrict__ poses, double* __restrict__ partials,
                int64_t* __restrict__ corr, const int32_t* __restrict__ exec_order) {
  __shared__ FactorShared sh;
  __shared__ double red[kWarps][kPartialStride];
  __shared__ double pose_s[24];
  constexpr int S = GVOX_LIN_STAGES;
  // the deep FAST pipeline (GVOX_LIN_DEEP) keeps, per warp, 2 stages of the
  // source A plane (64 float4), 2 of the B and N planes (128), 2 of the gathered
  // records' first two float4 per level (128 MAXL) and of their C_zz (16 MAXL)
  constexpr bool DEEP = GVOX_LIN_DEEP && GVOX_LIN_PIPE && !GVOX_LIN_BULK && FAST && ALL_DENSE && !VALID;
  constexpr int kDeepF4 = 64 + 128 + 128 * MAXL + 16 * MAXL;
  constexpr bool RPIPE = GVOX_LIN_RPIPE && !DEEP && GVOX_LIN_PIPE && !GVOX_LIN_BULK && FAST && ALL_DENSE && !VALID;
  constexpr int kWarpF4 = DEEP ? kDeepF4 : RPIPE ? 4 * 3 * 32 : S * 3 * 32;
  __shared__ __align__(128) float4 sbuf_raw[kWarps * kWarpF4];
  auto& sbuf = *reinterpret_cast<float4 (*)[kWarps][S][3][32]>(sbuf_raw);
  __shared__ __align__(8) uint64_t mbar[kWarps][S];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  // execution order -> tile (exec_order: the tiles grouped by target map, so
  // the CTAs resident together read the same target's grid and records; the
  // results do not depend on the order)
  const int64_t tile = exec_order ? (int64_t)__ldg(exec_order + blockIdx.x) : (int64_t)blockIdx.x;
  if (GVOX_LIN_BULK && lane == 0) {
#pragma unroll
    for (int j = 0; j < S; ++j) mbar_init(&mbar[warp][j], 1);
    fence_mbar_init();
  }
  stage_factor<MAXL>(sh, pose_s, clouds, maps, factors, tile_start, tile_factor, tile_pts, poses,
                     tile);
  const int L = FAST ? MAXL : sh.L;
  const int dyadic = FAST ? 1 : sh.dyadic;
  const double r0 = sh.r0, inv_r0 = sh.inv_r0;
  const float r0f = (float)sh.r0;
  // FAST: the visibility test only in the VALID instantiation
  const bool validate = FAST ? (VALID && sh.validate) : (bool)sh.validate;
  const bool error_only = sh.error_only;
  if (FAST) corr = nullptr;
  // 32-bit point index within the tile; the source planes pre-offset to its start
  const int64_t begin = sh.begin;
  const int32_t npts = (int32_t)(sh.end - sh.begin);
  int64_t* const corr_t = corr ? corr + sh.corr_base + begin * L : nullptr;
  Acc<MAXL> ac;

  const unsigned s_lane = smem_addr(&sbuf[warp][0][0][lane]);
  // prefetch of iteration i (points i * kThreads + 32 warp + lane) into stage st
  auto issue = [&](int32_t i, int st) {
    const int32_t base = i * kThreads + 32 * warp;
    if (GVOX_LIN_BULK) {
      // the warp's 32 points are one layout chunk: one 1536 B copy (a partial
      // last chunk copies its unused slots too, inside the allocation)
      if (lane == 0 && base < npts) {
        uint64_t* bar = &mbar[warp][st];
        mbar_expect_tx(bar, (unsigned)sizeof(sbuf[0][0]));
        bulk_g2s(&sbuf[warp][st][0][0], sh.A + (base >> 5) * 96, (unsigned)sizeof(sbuf[0][0]), bar);
      }
    } else {
      // each thread copies (and later reads) only its own slots: no warp sync
      if (base + lane < npts) {
        const unsigned sa = s_lane + (unsigned)st * (unsigned)sizeof(sbuf[0][0]);
        const float4* g = sh.A + ((base >> 5) * 96 + lane);
        cp_async16_s(sa, g);
        cp_async16_s(sa + 512u, g + 32);
        cp_async16_s(sa + 1024u, g + 64);
      }
      cp_async_commit();
    }
  };
#if GVOX_LIN_PIPE && !GVOX_LIN_BULK
  if constexpr (FAST) {
    // Software pipeline over points (FAST only): the next point is transformed
    // and its grid probes issued before the current point's voxel records are
    // gathered, so the two dependent memory round trips of consecutive points
    // overlap.  Needs a 3-stage ring: current (B, C planes), next (A plane),
    // and the copy in flight.
    static_assert(S == 3, "GVOX_LIN_PIPE uses a 3-stage ring");
    // Exact chunk culling (k_common.cuh chunk_culled_grid): iteration i of warp
    // w covers tile chunk 4 i + w; a chunk whose transformed box meets no
    // occupied coarsest-level cell has no correspondence at any level.  The warp
    // walks only its LIVE iterations (identical results: culled points add
    // nothing), so culled chunks are neither copied nor touched.
    constexpr int kMaxIters = GVOX_TILE_MAX_PPT * 256 / kThreads;  // iterations per warp
    static_assert(kMaxIters < 65535, "live iteration list holds 16-bit indices");
    constexpr int kNone = 0xFFFF;  // list padding: past every thread's last iteration
    __shared__ uint16_t live_s[kWarps][kMaxIters + 3];
    const int32_t iters = (npts - 32 * warp + kThreads - 1) / kThreads;
    const MapLevelDev& cv = sh.lv[MAXL - 1];
    // (no culling when validating: discarded points are counted, culled or not)
    const bool cull_on = GVOX_LIN_CULL && sh.cbox != nullptr && cv.grid != nullptr && !validate;
    // the warp's LIVE iterations, compacted in order into live_s[warp][0 .. nlive)
    int32_t nlive = 0;
#if GVOX_CULL_PREFETCH
    // the next pass's chunk box is loaded (3 x 8 B: boxes are 24 B apart) while
    // this pass's cells are tested
    auto load_box = [&](int32_t i, float2 (&b)[3]) {
      if (cull_on && i < iters) {
        const float2* bx = reinterpret_cast<const float2*>(sh.cbox + 6 * (i * kWarps + warp));
#pragma unroll
        for (int j = 0; j < 3; ++j) b[j] = __ldg(bx + j);
      }
    };
    float2 bnext[3];
    load_box(lane, bnext);
#pragma unroll 1
    for (int i0 = 0; i0 < iters; i0 += 32) {
      const int32_t i = i0 + lane;
      bool live = i < iters;
      const float box[6] = {bnext[0].x, bnext[0].y, bnext[1].x, bnext[1].y, bnext[2].x, bnext[2].y};
      load_box(i + 32, bnext);
      if (cull_on && live) live = !chunk_culled_grid(box, sh.Rf, sh.t, cv);
      const uint32_t m = __ballot_sync(0xffffffffu, live);
      if (live) live_s[warp][nlive + __popc(m & ((1u << lane) - 1u))] = (uint16_t)i;
      nlive += __popc(m);
    }
#else
#pragma unroll 1
    for (int i0 = 0; i0 < iters; i0 += 32) {
      const int32_t i = i0 + lane;
      bool live = i < iters;
      if (cull_on && live) {
        const float* bx = sh.cbox + 6 * (i * kWarps + warp);
        float box[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) box[j] = __ldg(bx + j);
        live = !chunk_culled_grid(box, sh.Rf, sh.t, cv);
      }
      const uint32_t m = __ballot_sync(0xffffffffu, live);
      if (live) live_s[warp][nlive + __popc(m & ((1u << lane) - 1u))] = (uint16_t)i;
      nlive += __popc(m);
    }
#endif
    if (lane < 3) live_s[warp][nlive + lane] = (uint16_t)kNone;  // the pipeline reads up to j + 3
    __syncwarp();
    const uint16_t* live_w = live_s[warp];
    auto live_at = [&](int32_t j) -> int32_t { return (int32_t)live_w[j]; };
    // this thread's point exists in iteration i  <=>  i < my_iters (kNone never)
    const int32_t my_iters = npts > tid ? (npts - tid + kThreads - 1) / kThreads : 0;
    // Per-thread copy addresses: iteration i of this warp is tile chunk
    // i * kWarps + warp, i.e. a fixed stride from the warp's first chunk; this
    // lane's slots of stage s sit at s_lane + s * (one stage).
    const float4* const g_lane = sh.A + (warp * 96 + lane);
    constexpr int kChunkStride = kWarps * 96;  // float4 per iteration
    constexpr unsigned kStageBytes = (unsigned)sizeof(sbuf[0][0]);
#if GVOX_LIN_DEEP
    if constexpr (DEEP) {
      // Three points deep, per thread (no warp barrier: each thread copies and
      // reads only its own slots).  Live iteration j, with X = point j,
      // Y = point j + 1, Z = point j + 2:
      //   wait for group j - 1 = {A plane of j + 2, B/N planes of j, records of j}
      //   prep Z: transform from its A plane, level-0 key, the three grid probes
      //   group j = {A plane of j + 3, B/N planes of Y, Y's voxel records (its
      //             probes landed during the previous point)} -> shared memory
      //   X's level terms and fold from shared memory
      // so a record gather has a whole point's work to land (the two-point
      // register pipeline consumed it right after issuing it).  Same arithmetic
      // in the same order as the other pipelines (bitwise equal, tested).
      struct DP {
        float qx, qy, qz, ex, ey, ez, cxx;
        uint32_t kb;  // low 24 bits: PointData::kb; bits 24 + l: level l has a voxel
        int32_t v[MAXL];
      };
      float4* const wbuf = sbuf_raw + warp * kDeepF4;
      const unsigned sw = smem_addr(wbuf) + 16u * (unsigned)lane;
      const unsigned sA = sw, sBN = sw + 64u * 16u, sG = sw + 192u * 16u;
      const unsigned sG2 = smem_addr(wbuf + 192 + 128 * MAXL) + 4u * (unsigned)lane;
      const float4* const rA = wbuf + lane;
      const float4* const rBN = wbuf + 64 + lane;
      const float4* const rG = wbuf + 192 + lane;
      const float* const rG2 = reinterpret_cast<const float*>(wbuf + 192 + 128 * MAXL) + lane;
      auto copy_a = [&](int32_t i, int s) {
        if (i < my_iters) cp_async16_s(sA + 512u * (unsigned)s, g_lane + i * kChunkStride);
      };
      auto copy_bn = [&](int32_t i, int s) {
        if (i < my_iters) {
          const float4* g = g_lane + i * kChunkStride;
          cp_async16_s(sBN + 1024u * (unsigned)s, g + 32);
          cp_async16_s(sBN + 1024u * (unsigned)s + 512u, g + 64);
        }
      };
      // Y's records: every level's, a miss (index -1) from the level's all-zero
      // sentinel record; nothing when Y hits no level (or has no point)
      auto gather = [&](DP& y, int s) {
        uint32_t hits = 0;
#pragma unroll
        for (int l = 0; l < MAXL; ++l) hits |= (y.v[l] >= 0 ? 1u : 0u) << l;
        y.kb |= hits << 24;
        if (hits) {
#pragma unroll
          for (int l = 0; l < MAXL; ++l) {
            const float4* vp = sh.lv[l].vox + 3 * y.v[l];
            const unsigned g = sG + (unsigned)(s * MAXL + l) * 1024u;
            cp_async16_ca(g, vp);
            cp_async16_ca(g + 512u, vp + 1);
            cp_async4_ca(sG2 + (unsigned)(s * MAXL + l) * 128u, &vp[2].x);
          }
        }
      };
      auto prep = [&](int32_t i, int s, DP& z) {
#pragma unroll
        for (int l = 0; l < MAXL; ++l) z.v[l] = -1;
        z.kb = 0;
        if (i < my_iters) {
          const float4 a = rA[32 * s];
          PointData pd;
          transform_point(sh, a, 1, r0, inv_r0, r0f, pd);
          lookup_nested<MAXL>(sh.lv, pd.k0x, pd.k0y, pd.k0z, z.v);
          z.qx = pd.qx;
          z.qy = pd.qy;
          z.qz = pd.qz;
          z.ex = pd.ex;
          z.ey = pd.ey;
          z.ez = pd.ez;
          z.kb = pd.kb;
          z.cxx = a.w;
        }
      };
      auto compute = [&](const DP& x, int s) {
        const uint32_t hits = x.kb >> 24;
        if (!hits) return;
        PointData q;
        q.qx = x.qx;
        q.qy = x.qy;
        q.qz = x.qz;
        q.ex = x.ex;
        q.ey = x.ey;
        q.ez = x.ez;
        q.kb = x.kb;
        const float4 b = rBN[64 * s], c = rBN[64 * s + 32];
        rcr(sh.Rf, sh.Rp, make_float4(0.f, 0.f, 0.f, x.cxx), b, c, q);
        LevelSum ls;
        ls.Oa = ls.Oc = ls.G = 0;
        ls.o11 = ls.o22 = ls.gz = 0.f;
        float bx = q.ex, by = q.ey, bz = q.ez;
#pragma unroll
        for (int l = 0; l < MAXL; ++l) {
          const float4 v0 = rG[(s * MAXL + l) * 64], v1 = rG[(s * MAXL + l) * 64 + 32];
          const float v2 = rG2[(s * MAXL + l) * 32];
          level_base(q, l, r0f, bx, by, bz);
          level_term<MAXL>(ac, ls, q, v0, v1, v2, l, bx, by, bz, (hits >> l) & 1u);
        }
        if (!error_only) fold_point<MAXL>(ac, ls, q);
      };
      // live iteration j (X, Y, Z as above; stage of point k = k & 1)
      int32_t i_n1 = live_at(1), i_n2 = live_at(2);
      auto step = [&](int32_t j, const DP& X, DP& Y, DP& Z) {
        cp_async_wait<0>();
        const int sj = j & 1;
        const int32_t i1 = i_n1, i2 = i_n2, i3 = live_at(j + 3);
        prep(i2, sj, Z);
        copy_a(i3, sj ^ 1);
        copy_bn(i1, sj ^ 1);
        gather(Y, sj ^ 1);
        cp_async_commit();
        compute(X, sj);
        i_n1 = i2;
        i_n2 = i3;
      };
      DP P0, P1, P2;
      {
        const int32_t i0 = live_at(0);
        copy_a(i0, 0);
        copy_a(i_n1, 1);
        cp_async_commit();
        cp_async_wait<0>();
        prep(i0, 0, P0);
        prep(i_n1, 1, P1);
        // group -1 = {A plane of point 2, B/N planes and records of point 0}
        copy_a(i_n2, 0);
        copy_bn(i0, 0);
        gather(P0, 0);
        cp_async_commit();
      }
#pragma unroll 1
      for (int32_t j = 0; j < nlive; j += 3) {
        step(j, P0, P1, P2);
        if (j + 1 >= nlive) break;
        step(j + 1, P1, P2, P0);
        if (j + 2 >= nlive) break;
        step(j + 2, P2, P0, P1);
      }
      cp_async_wait<0>();
      tile_reduce<MAXL>(ac, red, partials, tile);
      return;
    } else
#endif
#if GVOX_LIN_RPIPE
    if constexpr (RPIPE) {
      // Register pipeline, per thread.  Live iteration j (X = point j, Y = j + 1,
      // Z = j + 2; source stage of point k = k & 3):
      //   copy point j + 3's source planes (group j); wait for point j + 2's
      //   prep Z (transform, key, the three grid probes)
      //   gather Y's three voxel records into registers (its probes were issued
      //   one point ago)
      //   X's level terms and fold (its records were gathered one point ago)
      struct RP {
        float qx, qy, qz, ex, ey, ez;
        uint32_t kb;
        int32_t v[MAXL];
      };
      struct RR {
        float4 v0[MAXL], v1[MAXL];
        float v2[MAXL];
      };
      float4(*const rb)[3][32] = reinterpret_cast<float4(*)[3][32]>(sbuf_raw + warp * (4 * 3 * 32));
      const unsigned s_w = smem_addr(&rb[0][0][lane]);
      auto copy_src = [&](int32_t i, int s) {
        if (i < my_iters) {
          const float4* g = g_lane + i * kChunkStride;
          const unsigned sa = s_w + (unsigned)s * 1536u;
          cp_async16_s(sa, g);
          cp_async16_s(sa + 512u, g + 32);
          cp_async16_s(sa + 1024u, g + 64);
        }
        cp_async_commit();
      };
      auto prep = [&](int32_t i, int s, RP& z) {
#pragma unroll
        for (int l = 0; l < MAXL; ++l) z.v[l] = -1;
        if (i < my_iters) {
          const float4 a = rb[s][0][lane];
          PointData pd;
          transform_point(sh, a, 1, r0, inv_r0, r0f, pd);
          lookup_nested<MAXL>(sh.lv, pd.k0x, pd.k0y, pd.k0z, z.v);
          z.qx = pd.qx;
          z.qy = pd.qy;
          z.qz = pd.qz;
          z.ex = pd.ex;
          z.ey = pd.ey;
          z.ez = pd.ez;
          z.kb = pd.kb;
        }
      };
      // every level's record, a miss from the level's all-zero sentinel at -1
      auto gather = [&](const RP& y, RR& r) {
        bool any = false;
#pragma unroll
        for (int l = 0; l < MAXL; ++l) any |= y.v[l] >= 0;
        if (!any) return;  // (compute skips the point)
#pragma unroll
        for (int l = 0; l < MAXL; ++l) {
          const float4* vp = sh.lv[l].vox + 3 * y.v[l];
          r.v0[l] = __ldg(vp);
          r.v1[l] = __ldg(vp + 1);
          r.v2[l] = __ldg(&vp[2].x);
        }
      };
      auto compute = [&](const RP& x, const RR& r, int s) {
        bool any = false;
#pragma unroll
        for (int l = 0; l < MAXL; ++l) any |= x.v[l] >= 0;
        if (!any) return;
        PointData q;
        q.qx = x.qx;
        q.qy = x.qy;
        q.qz = x.qz;
        q.ex = x.ex;
        q.ey = x.ey;
        q.ez = x.ez;
        q.kb = x.kb;
        const float4 a = rb[s][0][lane], b = rb[s][1][lane], c = rb[s][2][lane];
        rcr(sh.Rf, sh.Rp, a, b, c, q);
        LevelSum ls;
        ls.Oa = ls.Oc = ls.G = 0;
        ls.o11 = ls.o22 = ls.gz = 0.f;
        float bx = q.ex, by = q.ey, bz = q.ez;
#pragma unroll
        for (int l = 0; l < MAXL; ++l) {
          level_base(q, l, r0f, bx, by, bz);
          level_term<MAXL>(ac, ls, q, r.v0[l], r.v1[l], r.v2[l], l, bx, by, bz, x.v[l] >= 0);
        }
        if (!error_only) fold_point<MAXL>(ac, ls, q);
      };
      int32_t i_n2 = live_at(2);  // before step j: live iteration j + 2
      auto step = [&](int32_t j, const RP& X, const RP& Y, RP& Z, const RR& RX, RR& RY) {
        const int32_t i3 = live_at(j + 3);
        copy_src(i3, (j + 3) & 3);
        cp_async_wait<1>();  // point j + 2's planes landed
        prep(i_n2, (j + 2) & 3, Z);
        gather(Y, RY);
        compute(X, RX, j & 3);
        i_n2 = i3;
      };
      RP P0, P1, P2;
      RR R0, R1;
      {
        const int32_t i0 = live_at(0), i1 = live_at(1);
        copy_src(i0, 0);
        copy_src(i1, 1);
        copy_src(i_n2, 2);
        cp_async_wait<1>();  // points 0 and 1 landed
        prep(i0, 0, P0);
        prep(i1, 1, P1);
        gather(P0, R0);
      }
#pragma unroll 1
      for (int32_t j = 0; j < nlive; j += 6) {
        step(j, P0, P1, P2, R0, R1);
        if (j + 1 >= nlive) break;
        step(j + 1, P1, P2, P0, R1, R0);
        if (j + 2 >= nlive) break;
        step(j + 2, P2, P0, P1, R0, R1);
        if (j + 3 >= nlive) break;
        step(j + 3, P0, P1, P2, R1, R0);
        if (j + 4 >= nlive) break;
        step(j + 4, P1, P2, P0, R0, R1);
        if (j + 5 >= nlive) break;
        step(j + 5, P2, P0, P1, R1, R0);
      }
      cp_async_wait<0>();
      tile_reduce<MAXL>(ac, red, partials, tile);
      return;
    } else
#endif
    {
    // the j-th live iteration's copy into stage j % S (one group per slot,
    // empty when the iteration does not exist or this lane has no point)
    auto issue_l = [&](int32_t i, unsigned sa) {
      if (i < my_iters) {
        const float4* g = g_lane + i * kChunkStride;
        cp_async16_s(sa, g);
        cp_async16_s(sa + 512u, g + 32);
        cp_async16_s(sa + 1024u, g + 64);
      }
      cp_async_commit();
    };
    int32_t i_cur = live_at(0);
    int32_t i_nxt = live_at(1);
    int32_t i_nx2 = live_at(2);
    issue_l(i_cur, s_lane);
    issue_l(i_nxt, s_lane + kStageBytes);
    cp_async_wait<S - 2>();  // the first live iteration landed
    // the current and the next point's transform, probe results and P:197
    // flag: two named sets whose roles alternate (GVOX_LIN_UNROLL2: the loop
    // is unrolled twice, so no register copy moves the next point's data into
    // the current one's)
    PointData pA, pB;
    int32_t vA[MAXL], vB[MAXL];
    bool invA = false, invB = false;
    auto prep = [&](int32_t i, int stg, PointData& pn, int32_t (&vn)[MAXL], bool& inv_n) {
#pragma unroll
      for (int l = 0; l < MAXL; ++l) vn[l] = -1;
      inv_n = false;
      if (i < my_iters) {
        const float4 a = sbuf[warp][stg][0][lane];
        if (VALID && validate && invisible(sh, a, sbuf[warp][stg][2][lane])) {
          inv_n = true;
          return;
        }
        transform_point(sh, a, 1, r0, inv_r0, r0f, pn);
        if (ALL_DENSE && GVOX_LIN_NESTED) {
          lookup_nested<MAXL>(sh.lv, pn.k0x, pn.k0y, pn.k0z, vn);
        } else if (ALL_DENSE) {
#pragma unroll
          for (int l = 0; l < MAXL; ++l)
            vn[l] = lookup_dense_pred(sh.lv[l], pn.k0x >> l, pn.k0y >> l, pn.k0z >> l);
        } else {
#pragma unroll
          for (int l = 0; l < MAXL; ++l)
            vn[l] = lookup_level<false>(sh.lv[l], pn.k0x >> l, pn.k0y >> l, pn.k0z >> l);
        }
      }
    };
    int st = 0;  // stage of the current live iteration
    // live iteration j: issue slot j + 2's copy, prepare point j + 1 (into the
    // other set), then this point's level terms and fold
    auto step = [&](int32_t j, const PointData& pd, const int32_t (&vid)[MAXL], const bool inv,
                    PointData& pn, int32_t (&vn)[MAXL], bool& inv_n) {
      bool any = false;
#pragma unroll
      for (int l = 0; l < MAXL; ++l) any |= vid[l] >= 0;
      // every level's record is loaded unconditionally: a level without a
      // correspondence (index -1) reads the level's all-zero sentinel record
      // at index -1 (masked out in level_term, exactly as zeros)
      float4 v0[MAXL], v1[MAXL];
      float v2[MAXL];
      auto gather = [&]() {
#pragma unroll
        for (int l = 0; l < MAXL; ++l) {
          const float4* vp = sh.lv[l].vox + 3 * vid[l];
          v0[l] = __ldg(vp);
          v1[l] = __ldg(vp + 1);
          v2[l] = __ldg(&vp[2].x);
        }
      };
      if (GVOX_LIN_ORDER == 2 && any && !(VALID && inv)) gather();
      issue_l(i_nx2, s_lane + (unsigned)(st == 0 ? S - 1 : st - 1) * kStageBytes);  // slot j + 2
      cp_async_wait<S - 2>();                                                        // slot j + 1 landed
      const int cur = st;
      if (++st == S) st = 0;
      prep(i_nxt, st, pn, vn, inv_n);
      i_cur = i_nxt;
      i_nxt = i_nx2;
      i_nx2 = live_at(j + 3);
      if (VALID && inv) {  // (only real points are marked)
        ++ac.n_invisible;
        return;
      }
      if (!any) return;  // (also every lane without a point: prep left its indices -1)
      PointData q = pd;  // (R C R^T lands in the point's record)
      if (GVOX_LIN_ORDER == 0) gather();
      {
        const float4 a = sbuf[warp][cur][0][lane], b = sbuf[warp][cur][1][lane],
                     c = sbuf[warp][cur][2][lane];
        rcr(sh.Rf, sh.Rp, a, b, c, q);
      }
      if (GVOX_LIN_ORDER == 1) gather();
      LevelSum ls;
      ls.Oa = ls.Oc = ls.G = 0;
      ls.o11 = ls.o22 = ls.gz = 0.f;
      float bx = q.ex, by = q.ey, bz = q.ez;
#pragma unroll
      for (int l = 0; l < MAXL; ++l) {
        level_base(q, l, r0f, bx, by, bz);
        level_term<MAXL>(ac, ls, q, v0[l], v1[l], v2[l], l, bx, by, bz, vid[l] >= 0);
      }
      if (!error_only) fold_point<MAXL>(ac, ls, q);
    };
    prep(i_cur, 0, pA, vA, invA);
#if GVOX_LIN_UNROLL2
#pragma unroll 1
    for (int32_t j = 0; j < nlive; j += 2) {
      step(j, pA, vA, invA, pB, vB, invB);
      if (j + 1 >= nlive) break;
      step(j + 1, pB, vB, invB, pA, vA, invA);
    }
#else
#pragma unroll 1
    for (int32_t j = 0; j < nlive; ++j) {
      step(j, pA, vA, invA, pB, vB, invB);
      pA = pB;
#pragma unroll
      for (int l = 0; l < MAXL; ++l) vA[l] = vB[l];
      invA = invB;
    }
#endif
    tile_reduce<MAXL>(ac, red, partials, tile);
    return;
    }
  }
#endif
#pragma unroll
  for (int j = 0; j < S - 1; ++j) issue(j, j);
  int st = 0, ph = 0;  // stage of iteration i and its mbarrier phase
  for (int32_t i = 0; i * kThreads + 32 * warp < npts; ++i) {
    if (GVOX_LIN_BULK) __syncwarp();  // all lanes done with the stage refilled below
    issue(i + S - 1, st == 0 ? S - 1 : st - 1);
    if (GVOX_LIN_BULK)
      mbar_wait(&mbar[warp][st], (unsigned)ph);
    else
      cp_async_wait<S - 1>();
    const int cur = st;
    if (++st == S) {
      st = 0;
      ph ^= 1;
    }
    const int32_t k = i * kThreads + 32 * warp + lane;
    if (k >= npts) continue;
    const float4 a = sbuf[warp][cur][0][lane], b = sbuf[warp][cur][1][lane],
                 c = sbuf[warp][cur][2][lane];
    if (!FAST && validate && invisible(sh, a, c)) {
      ++ac.n_invisible;
      if (corr)
        for (int l = 0; l < L; ++l) corr_t[k * L + l] = -2;
      continue;
    }
    PointData pd;
    transform_point(sh, a, dyadic, r0, inv_r0, r0f, pd);
    float bx = pd.ex, by = pd.ey, bz = pd.ez;  // residual base, advanced level by level
    bool have_rcr = false;
    LevelSum ls;
    ls.Oa = ls.Oc = ls.G = 0;
    ls.o11 = ls.o22 = ls.gz = 0.f;
    // levels are processed in groups of G (all loads of a group in flight together)
    constexpr int G = MAXL < GVOX_LIN_G ? MAXL : GVOX_LIN_G;
#pragma unroll
    for (int lb = 0; lb < MAXL; lb += G) {
      if (!FAST && lb >= L) break;
      int32_t vid[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int l = lb + j;
        if (FAST)
          vid[j] = lookup_dense_pred(sh.lv[l], pd.k0x >> l, pd.k0y >> l, pd.k0z >> l);
        else
          vid[j] = l < L ? lookup_level<ALL_DENSE>(sh.lv[l], pd.k0x >> l, pd.k0y >> l, pd.k0z >> l)
                         : -1;
      }
      if (corr) {
        for (int j = 0; j < G && lb + j < L; ++j) {
          const int l = lb + j;
          corr_t[k * L + l] =
              vid[j] >= 0 ? (int64_t)pack_key(pd.k0x >> l, pd.k0y >> l, pd.k0z >> l) : -1;
        }
      }
      bool any = false;
#pragma unroll
      for (int j = 0; j < G; ++j) any |= vid[j] >= 0;
      if (!any) {
#pragma unroll
        for (int j = 0; j < G; ++j)  // (the bases of the skipped levels still advance)
          if (lb + j > 0) level_base(pd, lb + j, r0f, bx, by, bz);
        continue;
      }
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
      if (!have_rcr) {
        have_rcr = true;
        rcr(sh.Rf, sh.Rp, a, b, c, pd);
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        if (lb + j > 0) level_base(pd, lb + j, r0f, bx, by, bz);
        if (vid[j] >= 0) level_term<MAXL>(ac, ls, pd, v0[j], v1[j], v2[j], lb + j, bx, by, bz);
      }
    }
    if (have_rcr && !error_only) fold_point<MAXL>(ac, ls, pd);
  }
  tile_reduce<MAXL>(ac, red, partials, tile);
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
  // fixed order (4 interleaved partial sums over the tiles, then combined) ->
  // deterministic; the 4 chains keep 4 loads in flight per lane
  for (int j = lane; j < kPartialStride; j += 32) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int32_t t = t0;
    for (; t + 4 <= t1; t += 4) {
      const double* q = partials + (int64_t)t * kPartialStride + j;
      s0 += q[0];
      s1 += q[kPartialStride];
      s2 += q[2 * kPartialStride];
      s3 += q[3 * kPartialStride];
    }
    for (; t < t1; ++t) s0 += partials[(int64_t)t * kPartialStride + j];
    sum_s[w][j] = (s0 + s1) + (s2 + s3);
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
                      bool all_dense, bool fast, bool validate, cudaStream_t stream,
                      const int32_t* exec_order) {
  if (num_tiles <= 0) return;
  const unsigned grid = (unsigned)num_tiles;
  // FAST (3 dyadic levels, no dump): dense grids or hash levels, with or
  // without the P:197 visibility test
  if (fast && max_levels == 3) {
    note_linearize_variant(GVOX_LINVAR_FAST | (all_dense ? GVOX_LINVAR_DENSE : 0) |
                           (validate ? GVOX_LINVAR_VALID : 0) | (3 << 8));
    auto* k = all_dense ? (validate ? k_linearize<3, true, true, true> : k_linearize<3, true, true, false>)
                        : (validate ? k_linearize<3, false, true, true> : k_linearize<3, false, true, false>);
    k<<<grid, kThreads, 0, stream>>>(clouds, maps, factors, tile_start, tile_factor, tile_pts, poses,
                                     partials, nullptr, exec_order);
  } else if (max_levels <= 3) {
    note_linearize_variant((all_dense ? GVOX_LINVAR_DENSE : 0) | (3 << 8));
    if (all_dense)
      k_linearize<3, true, false><<<grid, kThreads, 0, stream>>>(
          clouds, maps, factors, tile_start, tile_factor, tile_pts, poses, partials, corr_dump, exec_order);
    else
      k_linearize<3, false, false><<<grid, kThreads, 0, stream>>>(
          clouds, maps, factors, tile_start, tile_factor, tile_pts, poses, partials, corr_dump, exec_order);
  } else {
    note_linearize_variant(GVOX_MAX_LEVELS << 8);
    k_linearize<GVOX_MAX_LEVELS, false, false><<<grid, kThreads, 0, stream>>>(
        clouds, maps, factors, tile_start, tile_factor, tile_pts, poses, partials, corr_dump, exec_order);
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

// Device-side plan of a screened batch (gvox_linearize_batch_accum_select):
// compact the candidates whose selected[p] != 0, in candidate order, into
// factors_c[0..S), their tile starts tile_start_c[0..S] (tiles per candidate
// from the host plan, a function of the factor alone) and counts = {S, T}.
// Two coalesced passes of one thread per candidate: per-block totals, then
// each block's offset (sum of the earlier blocks' totals), a block scan and
// the scatter.
constexpr int kPlanThreads = 1024;

// inclusive block scan of (a, b) over the block's threads; returns the totals
__device__ __forceinline__ int2 block_scan2(int32_t& a, int32_t& b, int2* s_w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t xa = __shfl_up_sync(0xffffffffu, a, o), xb = __shfl_up_sync(0xffffffffu, b, o);
    if (lane >= o) {
      a += xa;
      b += xb;
    }
  }
  if (lane == 31) s_w[warp] = make_int2(a, b);
  __syncthreads();
  if (warp == 0) {
    int2 v = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t xa = __shfl_up_sync(0xffffffffu, v.x, o), xb = __shfl_up_sync(0xffffffffu, v.y, o);
      if (lane >= o) {
        v.x += xa;
        v.y += xb;
      }
    }
    s_w[lane] = v;  // inclusive warp-total prefix
  }
  __syncthreads();
  if (warp > 0) {
    a += s_w[warp - 1].x;
    b += s_w[warp - 1].y;
  }
  return s_w[31];
}

__global__ void __launch_bounds__(kPlanThreads)
    k_select_count(const uint8_t* __restrict__ selected, const int32_t* __restrict__ ntiles,
                   int64_t num_cand, int2* __restrict__ block_tot, int32_t* __restrict__ counts) {
  __shared__ int2 s_w[32];
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[2] = counts[3] = 0;  // (k_select_scatter reduces into them)
  const int64_t p = (int64_t)blockIdx.x * kPlanThreads + threadIdx.x;
  int32_t f = p < num_cand && selected[p] ? 1 : 0;
  int32_t t = f ? ntiles[p] : 0;
  const int2 tot = block_scan2(f, t, s_w);
  if (threadIdx.x == 0) block_tot[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kPlanThreads)
    k_select_scatter(const uint8_t* __restrict__ selected, const int32_t* __restrict__ ntiles,
                     const uint8_t* __restrict__ cls, const FactorDev* __restrict__ factors,
                     int64_t num_cand,
                     const int2* __restrict__ block_tot, FactorDev* __restrict__ factors_c,
                     int32_t* __restrict__ tile_start_c, int32_t* __restrict__ counts) {
  __shared__ int2 s_w[32];
  __shared__ int2 s_off;
  // this block's offset: the totals of the blocks before it
  int32_t of = 0, ot = 0;
  for (int j = threadIdx.x; j < (int)blockIdx.x; j += kPlanThreads) {
    const int2 v = block_tot[j];
    of += v.x;
    ot += v.y;
  }
  {
    int32_t a = of, b = ot;
    const int2 tot = block_scan2(a, b, s_w);
    if (threadIdx.x == 0) s_off = tot;
    __syncthreads();
  }
  const int2 off = s_off;
  const int64_t p = (int64_t)blockIdx.x * kPlanThreads + threadIdx.x;
  const bool sel = p < num_cand && selected[p];
  const int32_t nt = sel ? ntiles[p] : 0;
  int32_t f = sel ? 1 : 0, t = nt;
  const int2 tot = block_scan2(f, t, s_w);
  if (sel) {
    const int32_t k = off.x + f - 1;  // exclusive position
    factors_c[k] = factors[p];
    tile_start_c[k] = off.y + t - nt;
  }
  // kernel class of the selected candidates: OR of the class bits, max levels
  // (warp-aggregated, one atomic pair per warp with a selected candidate)
  const uint32_t c = sel ? (uint32_t)cls[p] : 0u;
  const uint32_t c_or = __reduce_or_sync(0xffffffffu, c & 15u);
  const uint32_t c_lv = __reduce_max_sync(0xffffffffu, c >> 4);
  if ((threadIdx.x & 31) == 0 && (c_or | c_lv)) {
    atomicOr(counts + 2, (int32_t)c_or);
    atomicMax(counts + 3, (int32_t)c_lv);
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    tile_start_c[off.x + tot.x] = off.y + tot.y;
    counts[0] = off.x + tot.x;
    counts[1] = off.y + tot.y;
  }
}

// ---- execution order of a screened batch's tiles, grouped by target map
// (counting sort on the device: tiles per target, an exclusive scan, then each
// factor's tiles scattered to its target's range; the order inside a target is
// whatever the atomics give -- execution order only, results unaffected)
__global__ void k_exec_count(const FactorDev* __restrict__ fc, const int32_t* __restrict__ tsc,
                             int64_t S, int32_t* __restrict__ hist) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f < S) atomicAdd(hist + fc[f].tgt, tsc[f + 1] - tsc[f]);
}
__global__ void __launch_bounds__(1024) k_exec_scan(int32_t* __restrict__ hist, int64_t n) {
  // one block: exclusive scan of n counts in chunks of 1024
  __shared__ int32_t s_w[32];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b = 0; b < n; b += 1024) {
    const int64_t i = b + threadIdx.x;
    const int32_t v = i < n ? hist[i] : 0;
    int32_t x = v;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      int32_t w = s_w[threadIdx.x];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= o) w += y;
      }
      s_w[threadIdx.x] = w;  // inclusive over warps
    }
    __syncthreads();
    const int32_t warp_off = (threadIdx.x >> 5) ? s_w[(threadIdx.x >> 5) - 1] : 0;
    const int32_t c = carry;
    if (i < n) hist[i] = c + warp_off + x - v;  // exclusive
    __syncthreads();
    if (threadIdx.x == 1023) carry = c + warp_off + x;
    __syncthreads();
  }
}
__global__ void k_exec_scatter(const FactorDev* __restrict__ fc, const int32_t* __restrict__ tsc,
                               int64_t S, int32_t* __restrict__ cursor, int32_t* __restrict__ exec) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= S) return;
  const int32_t t0 = tsc[f], nt = tsc[f + 1] - t0;
  const int32_t b = atomicAdd(cursor + fc[f].tgt, nt);
  for (int32_t k = 0; k < nt; ++k) exec[b + k] = t0 + k;
}

void launch_exec_order_by_target(const FactorDev* fc, const int32_t* tsc, int64_t S,
                                 int64_t num_maps, int32_t* hist, int32_t* exec,
                                 cudaStream_t stream) {
  if (S <= 0) return;
  cudaMemsetAsync(hist, 0, 4 * (size_t)num_maps, stream);
  const unsigned nb = (unsigned)((S + 255) / 256);
  k_exec_count<<<nb, 256, 0, stream>>>(fc, tsc, S, hist);
  note_launch();
  k_exec_scan<<<1, 1024, 0, stream>>>(hist, num_maps);
  note_launch();
  k_exec_scatter<<<nb, 256, 0, stream>>>(fc, tsc, S, hist, exec);
  note_launch();
}

void launch_select_plan(const uint8_t* selected, const int32_t* ntiles, const uint8_t* cls,
                        const FactorDev* factors, int64_t num_cand, FactorDev* factors_c,
                        int32_t* tile_start_c, int32_t* counts, int2* block_tot,
                        cudaStream_t stream) {
  const unsigned nb = (unsigned)((num_cand + kPlanThreads - 1) / kPlanThreads);
  k_select_count<<<nb, kPlanThreads, 0, stream>>>(selected, ntiles, num_cand, block_tot, counts);
  note_launch();
  k_select_scatter<<<nb, kPlanThreads, 0, stream>>>(selected, ntiles, cls, factors, num_cand,
                                                    block_tot, factors_c, tile_start_c, counts);
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
