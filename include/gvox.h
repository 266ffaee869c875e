/*
 * gvox.h -- C ABI of the B200-native batched VGICP linearization library
 * (libgvox.so), the data-parallel hot path of GLIM (arXiv 2407.10344).
 *
 * Citations: "P:n" = PAPER.md line n of the paper's source (Sec. III-C
 * "Matching Cost Factor": Preprocessing P:186, Correspondence search P:197,
 * Linearization P:199-218 = Eqs. 2-8, Implementation P:221-224 / Fig. 4
 * P:190-195; overlap rate P:280; global factor selection P:391).  Readings of
 * ambiguous passages (Q1..Q19) are listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Poses are fp64, row-major 3x4 [R | t], world <- sensor.  The relative
 *    pose of a factor is T_ij = T_j^-1 T_i (source cloud i, target map j;
 *    reading Q1).  Tangent vectors are rotation-first [w; rho]; perturbations
 *    are right-multiplied, T <- T Exp(xi).
 *  - Covariances are 6 floats per point: xx, xy, xz, yy, yz, zz.
 *  - Voxel level l (0-based) has resolution r_l = r0 * 2^l (P:186, 1-based
 *    there).  A voxel key is floor(p / r_l) per axis, evaluated in fp64 from
 *    the fp32 input promoted exactly (reading Q10); it is identified by the
 *    packed key ((kx+2^20)<<42) | ((ky+2^20)<<21) | (kz+2^20), valid for
 *    -2^20 <= k < 2^20 (reading Q11).
 *  - Every call enqueues its work on the context's CUDA stream.  Calls whose
 *    outputs are host memory (mem == GVOX_HOST) synchronize that stream before
 *    returning; calls with device outputs do not.
 *  - Status codes only; no exception crosses the ABI.  On failure
 *    gvox_last_error() returns a thread-local message naming the offending
 *    argument (for factors: the factor index).
 *  - Not thread-safe per context: one host thread drives one gvox_ctx.
 */
#ifndef GVOX_H_
#define GVOX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GVOX_VERSION_MAJOR 0
#define GVOX_VERSION_MINOR 1
#define GVOX_MAX_LEVELS 8

typedef enum gvox_status {
  GVOX_OK = 0,
  GVOX_ERR_INVALID = 1, /* null pointer, bad size, r0 <= 0 or non-finite, levels
                           outside [1, 8], index out of range, non-finite input */
  GVOX_ERR_RANGE = 2,   /* a voxel key outside [-2^20, 2^20) during a map build */
  GVOX_ERR_CUDA = 3,    /* CUDA runtime error (message has cudaGetErrorString) */
  GVOX_ERR_NOMEM = 4    /* device or pinned host allocation failed */
} gvox_status;

/* Where a caller-provided buffer lives. */
enum { GVOX_HOST = 0, GVOX_DEVICE = 1 };

/* Per-factor flags. */
enum {
  /* P:197 surface-orientation validation: discard point k at every level when
     (mu_k - T_i^-1 t_j) . n_k > 0 (strict; a zero normal disables it, Q7).
     Needs normals oriented toward the source sensor origin. */
  GVOX_F_VALIDATE_SURFACE = 1u,
  /* Error and counts only; H and b are left zero (LM trial steps). */
  GVOX_F_ERROR_ONLY = 2u
};

typedef struct gvox_ctx gvox_ctx;
typedef struct gvox_cloud gvox_cloud;
typedef struct gvox_map gvox_map;

/* One matching cost factor: indices into the clouds[], maps[] and poses[]
   arrays of the call. */
typedef struct gvox_factor {
  int32_t source_cloud; /* P_i, points in frame i */
  int32_t target_map;   /* voxelmap of P_j, in frame j */
  int32_t pose_i;       /* linearization point T_i */
  int32_t pose_j;       /* linearization point T_j */
  uint32_t flags;       /* GVOX_F_* */
} gvox_factor;

/* One overlap query: source cloud P_i against the voxels of P_j. */
typedef struct gvox_pair {
  int32_t source_cloud;
  int32_t target_map;
  int32_t pose_i;
  int32_t pose_j;
} gvox_pair;

/* Linearized factor (Eqs. 4-8), blocks over (x_i, x_j):
     H_ii = sum A^T Omega A, H_ij = sum A^T Omega B, H_jj = sum B^T Omega B,
     b_i  = sum A^T Omega d,  b_j  = sum B^T Omega d,  error = sum d^T Omega d
   with d = mu~ - T_ij mu, A = [R_ij (mu)x, -R_ij], B = [-(T_ij mu)x, I]
   (readings Q2-Q5: sums over points and levels, no 1/2, b as printed).
   Matrices are row-major 6x6.  e(delta) ~ error + 2 b^T delta + delta^T H delta;
   the Gauss-Newton step is -H^-1 b. */
typedef struct gvox_linear_factor {
  double H_ii[36];
  double H_ij[36];
  double H_jj[36];
  double b_i[6];
  double b_j[6];
  double error;
  int32_t inliers[GVOX_MAX_LEVELS]; /* correspondences found per level */
  int32_t num_invisible;            /* points discarded by validation */
  int32_t num_degenerate;           /* terms skipped: fused covariance not PD (Q16) */
} gvox_linear_factor;

/* Compact per-factor result in target-block form, 288 bytes: what one rank
   contributes to the multi-GPU gather.  terms[0..20] = upper triangle of H_jj
   (row-major), terms[21..26] = b_j, terms[27] = error.  gvox_expand() turns it
   into a gvox_linear_factor via H_ii = Ad^T H_jj Ad, H_ij = -Ad^T H_jj,
   b_i = -Ad^T b_j with Ad = Ad(T_ij) (exact: A = -B Ad(T_ij)). */
typedef struct gvox_factor_accum {
  double terms[28];
  int32_t inliers[GVOX_MAX_LEVELS];
  int32_t num_invisible;
  int32_t num_degenerate;
  int32_t reserved[6];
} gvox_factor_accum;

/* ---------------------------------------------------------------- context */

/* Create a context on CUDA device `device`, enqueuing on `cuda_stream`
   (a cudaStream_t; NULL = the legacy default stream).  The stream is not owned. */
gvox_status gvox_ctx_create(int device, void* cuda_stream, gvox_ctx** out);
/* Move the context to another stream.  The new stream is first ordered after
   everything already enqueued on the old one (an event), so the context's
   reused workspaces never race across the switch. */
gvox_status gvox_ctx_set_stream(gvox_ctx* ctx, void* cuda_stream);
void gvox_ctx_destroy(gvox_ctx* ctx);

/* Device-side timing of the library's own kernels.  When enabled, every launch
   of a kernel group is bracketed by CUDA events on the context stream;
   gvox_ctx_timing() (synchronizes) returns the summed elapsed milliseconds and
   the launch count per group, optionally resetting them.  ms and launches are
   arrays of GVOX_TIMER_COUNT entries (either may be NULL). */
enum {
  GVOX_TIMER_BUILD = 0,     /* voxelmap insert / accumulate / finalize kernels */
  GVOX_TIMER_OVERLAP = 1,   /* overlap kernel */
  GVOX_TIMER_LINEARIZE = 2, /* fused correspondence + linearization kernel */
  GVOX_TIMER_REDUCE = 3,    /* per-factor reduction / expansion kernel */
  GVOX_TIMER_REGISTER = 4,  /* one gvox_register_batch graph launch (all iterations) */
  GVOX_TIMER_PREPROCESS = 5, /* k-NN (count, scan, scatter, query) / covariance kernels */
  GVOX_TIMER_SOLVE = 6,     /* gvox_solve_global: expand, assemble, PCG, scatter */
  GVOX_TIMER_COUNT = 7
};
gvox_status gvox_ctx_enable_timing(gvox_ctx* ctx, int enable);
gvox_status gvox_ctx_timing(gvox_ctx* ctx, double* ms, int64_t* launches, int reset);

/* ----------------------------------------------------------------- clouds */

/* Gaussian point cloud (p_k = (mu_k, C_k)), optionally with normals for
   the P:197 validation.  mu: n x 3 floats, cov: n x 6 floats, normals: n x 3
   floats or NULL.  mem selects where the three arrays live (all the same).
   The data are copied into a device-resident, library-owned handle (planar
   float4 layout), so the caller may free its arrays after return.
   Errors: GVOX_ERR_INVALID for null pointers (with n > 0), n < 0, or a
   non-finite coordinate / covariance / normal (this call synchronizes). */
gvox_status gvox_cloud_create(gvox_ctx* ctx, const float* mu, const float* cov,
                              const float* normals, int64_t n, int mem, gvox_cloud** out);
/* Batched creation of `count` clouds stored back to back: cloud k holds points
   [offsets[k], offsets[k+1]) of mu / cov / normals (offsets: host int64
   [count + 1], offsets[0] = 0).  One copy, one packing launch and one
   synchronization for the whole set; the clouds share one device allocation
   (freed when the last of them is destroyed). */
gvox_status gvox_clouds_create(gvox_ctx* ctx, const float* mu, const float* cov,
                               const float* normals, const int64_t* offsets, int64_t count,
                               int mem, gvox_cloud** clouds_out);
int64_t gvox_cloud_size(const gvox_cloud* cloud);
void gvox_cloud_destroy(gvox_cloud* cloud);

/* -------------------------------------------------------------- voxelmaps */

/* Multi-resolution Gaussian voxelmap of a cloud: for each level
   l < levels, voxels keyed by floor(mu / r_l); each voxel holds the mean of
   its points' means, the mean of their covariances and the point count
   (reading Q9).  Built on the device by spatial hashing.
   Errors: GVOX_ERR_INVALID (r0 <= 0 or non-finite, levels outside [1, 8]),
   GVOX_ERR_RANGE (some key outside [-2^20, 2^20) at some level).
   Synchronizes once (to size the voxel arrays). */
gvox_status gvox_create_voxelmap(gvox_ctx* ctx, const gvox_cloud* cloud, double r0, int levels,
                                 gvox_map** out);

/* Batched build of `count` maps with one launch sequence (same r0, levels).
   maps_out[k] receives the map of clouds[k].  All-or-nothing on error. */
gvox_status gvox_create_voxelmaps(gvox_ctx* ctx, const gvox_cloud* const* clouds, int64_t count,
                                  double r0, int levels, gvox_map** maps_out);

gvox_status gvox_voxelmap_info(const gvox_map* map, int level, int64_t* num_voxels,
                               double* resolution);
int gvox_voxelmap_levels(const gvox_map* map);

/* Canonical export of one level to HOST arrays, voxels in ascending packed-key
   order: keys [V], means [V x 3] (fp64 = centre + stored fp32 offset),
   covs [V x 6], counts [V].  Any output pointer may be NULL.  Synchronizes. */
gvox_status gvox_voxelmap_export(gvox_ctx* ctx, const gvox_map* map, int level, int64_t* keys,
                                 double* means, double* covs, int32_t* counts);

/* Lookup: for n query points q (fp64, n x 3, in the map frame),
   the packed key of the containing voxel at `level`, or -1 if that voxel is
   empty or out of key range (no neighbour search, reading Q8).
   q and keys_out live in `mem`. */
gvox_status gvox_voxelmap_lookup(gvox_ctx* ctx, const gvox_map* map, int level, const double* q,
                                 int64_t n, int64_t* keys_out, int mem);

void gvox_map_destroy(gvox_map* map);
/* Destroy count maps (NULL entries skipped) in one call: what a caller that
   built a batch with gvox_create_voxelmaps does once the batch is done (the
   per-call overhead of one destroy per map shows in odometry-sized steps). */
void gvox_maps_destroy(gvox_map* const* maps, int64_t count);

/* ---------------------------------------------------------------- overlap */

/* Overlap counts ("the fraction of points in P_i that fall within a
   voxel of P_j"): counts[p] = number of points of clouds[pairs[p].source_cloud]
   whose key under T_ij = T_j^-1 T_i (fp64, pinned fma order) is occupied at
   `level` of maps[pairs[p].target_map].  No validation (reading Q15).  The
   rate is counts[p] / n (0 for an empty source); the global-mapping factor
   test "exceeds 5 %" is 20 * count > n.
   pairs, poses: host arrays.  counts: int32 [num_pairs] in `mem`.
   Exactly one H2D (pairs + poses) per call; one D2H when mem == GVOX_HOST. */
gvox_status gvox_overlap(gvox_ctx* ctx, const gvox_cloud* const* clouds, int64_t num_clouds,
                         const gvox_map* const* maps, int64_t num_maps, const gvox_pair* pairs,
                         int64_t num_pairs, const double* poses, int64_t num_poses, int level,
                         int32_t* counts, int mem);

/* Screening decision for factor creation ("a matching cost factor
   between each submap pair with an overlap rate that exceeds a small threshold
   (e.g., 5 %)"): selected[p] = 1 iff count * den > n * num, with count and n as
   in gvox_overlap (e.g. num = 1, den = 20 for "exceeds 5 %").  Every pair stops
   as soon as its decision is certain (enough hits, or too few points left), so
   the decision is exactly the one the full count gives with fewer lookups.
   num >= 0, den > 0.  selected: uint8 [num_pairs] in `mem`.  Same transfers as
   gvox_overlap. */
gvox_status gvox_overlap_select(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                int64_t num_clouds, const gvox_map* const* maps, int64_t num_maps,
                                const gvox_pair* pairs, int64_t num_pairs, const double* poses,
                                int64_t num_poses, int level, int32_t num, int32_t den,
                                uint8_t* selected, int mem);

/* ---------------------------------------------------------- preprocessing */

/* Exact k nearest neighbours ("C_k is calculated from neighboring
   points of p_k given by a k-nearest-neighbor search"; "the costly
   exact nearest neighbor search is only performed in the preprocessing
   step").  A batch of `count` independent clouds stored back to back:
   cloud c = points [offsets[c], offsets[c+1]) of `points` (n x 3 floats).
   neighbors (n x k int32): row i lists the k points of i's cloud nearest to i
   (self included) as LOCAL indices within the cloud, ordered by (squared
   distance, index) ascending; -1 pads rows of clouds with fewer than k
   points.  Distances: fp64 d2 = (dx*dx + dy*dy) + dz*dz from the fp32 inputs
   with no fused multiply-add (reading R26), so the result is unique.
   cell_size (> 0, metres): the search grid pitch; speed only, never the
   result (about twice the downsampling resolution works well).
   1 <= k <= 32.  offsets: host int64 [count + 1], offsets[0] = 0.  points and
   neighbors live in `mem`.  Synchronizes once (to size the grids).
   Errors: GVOX_ERR_INVALID for bad sizes or a non-finite coordinate. */
gvox_status gvox_knn(gvox_ctx* ctx, const float* points, const int64_t* offsets, int64_t count,
                     int32_t k, double cell_size, int32_t* neighbors, int mem);

/* Per-point covariance from a neighbour table (reading R27): the
   sample covariance of the point's neighbours (fp64), the unit eigenvector n
   of its smallest eigenvalue oriented toward the cloud origin (n . mu <= 0),
   and the GICP plane model C = I - (1 - 1e-3) n n^T (eigenvalues 1e-3, 1, 1).
   A zero sample covariance gives C = 1e-6 I and n = 0 (R28).  neighbors as
   produced by gvox_knn (local indices, -1 = none; other values are rejected
   for host arrays and undefined behaviour for device arrays).  cov (n x 6:
   xx xy xz yy yz zz) and normals (n x 3) are fp32 in `mem`, like points and
   neighbors.  The neighbour table may come from an earlier pose of the same
   points (reused after deskewing). */
gvox_status gvox_estimate_covariances(gvox_ctx* ctx, const float* points, const int64_t* offsets,
                                      int64_t count, const int32_t* neighbors, int32_t k,
                                      float* cov, float* normals, int mem);

/* ------------------------------------------------------------- keyframes */

/* Overlap with a UNION of maps ("we evaluate the overlap rate between
   that frame and the union of all keyframes, and if the overlap is smaller
   than a threshold (e.g., 90%), we insert that frame into the keyframe
   list").  Query q: counts[q] = number of points of clouds[queries[q].source_cloud]
   at pose queries[q].pose_i whose key at `level` is occupied in AT LEAST ONE
   of the maps members[first .. first + count) (each at its own pose_j; keys
   and poses as in gvox_overlap).  The rate is counts[q] / n; the insertion
   test "smaller than 90 %" is 10 * count < 9 * n.  count = 0 gives 0.
   queries, members, poses: host arrays; counts: int32 [num_queries] in `mem`.
   One H2D; one D2H when mem == GVOX_HOST. */
typedef struct gvox_union_query {
  int32_t source_cloud;
  int32_t pose_i;
  int32_t first; /* into members[] */
  int32_t count; /* >= 0 */
} gvox_union_query;
typedef struct gvox_union_member {
  int32_t target_map;
  int32_t pose_j;
} gvox_union_member;
gvox_status gvox_overlap_union(gvox_ctx* ctx, const gvox_cloud* const* clouds, int64_t num_clouds,
                               const gvox_map* const* maps, int64_t num_maps,
                               const gvox_union_query* queries, int64_t num_queries,
                               const gvox_union_member* members, int64_t num_members,
                               const double* poses, int64_t num_poses, int level,
                               int32_t* counts, int mem);

/* Keyframe removal rule (host only, no GPU work).  Keyframes
   0 .. K-1 in list order, K-1 = the latest keyframe; overlap[i * K + j] =
   o(i, j), the overlap rate of keyframe i's points in keyframe j's voxels
   (gvox_overlap counts / n_i).  remove[i] (K bytes out) is set to 1 for
     1. every i < K-1 with o(i, K-1) < min_overlap ("overlap the latest
        keyframe by less than a certain threshold (e.g., 5%)");
     2. then, if more than n_odom keyframes remain, the ONE remaining i < K-1
        minimising s(i) = o(i, K-1) * sum_{j remaining, j != i, j < K-1} (1 - o(i, j))
        (ties: the smallest i).  Reading R25: the paper's
        j in [1, N_odom - 1] \ {i} is every other non-latest keyframe.
   The latest keyframe is never removed.  K >= 1, n_odom >= 1. */
gvox_status gvox_keyframe_update(const double* overlap, int32_t K, int32_t n_odom,
                                 double min_overlap, uint8_t* remove);

/* Keyframe insertion test (host only): "if the overlap [of the new
   frame with the union of all keyframes] is smaller than a threshold (e.g.,
   90%), we insert that frame".  count: gvox_overlap_union's count for the
   frame (points of the frame inside a voxel of any keyframe), n: the frame's
   point count.  The rate count / n is compared in integers,
   insert = (den * count < num * n) (default num / den = 9 / 10; strict
   "smaller than").  An empty keyframe list is the caller's case (always
   insert); n = 0 gives 0 < 0, false: an empty frame adds nothing and is not
   inserted (the oracle's rule, oracle/keyframes.py).  GVOX_ERR_INVALID for count < 0,
   n < 0, count > n, num < 0, den <= 0 or a NULL output. */
gvox_status gvox_keyframe_insert_test(int64_t count, int64_t n, int32_t num, int32_t den,
                                      int32_t* insert);

/* The removal rule of gvox_keyframe_update from raw gvox_overlap COUNTS (P:280
   "overlap rate between frames": the fraction of keyframe i's points that fall
   within a voxel of keyframe j): counts[i * K + j] = points of keyframe i in
   keyframe j's voxels, sizes[i] = keyframe i's point count, K-1 = the latest
   keyframe.  o(i, j) = counts / sizes[i] (0 for an empty keyframe) is formed
   here, in fp64, then the rules apply exactly as gvox_keyframe_update.
   overlap_out (optional, K * K doubles): the o(i, j) matrix used.
   GVOX_ERR_INVALID for negative counts or sizes, counts[i*K+j] > sizes[i]. */
gvox_status gvox_keyframe_update_counts(const int64_t* counts, const int64_t* sizes, int32_t K,
                                        int32_t n_odom, double min_overlap, uint8_t* remove,
                                        double* overlap_out);

/* ------------------------------------------------------------- linearize */

/* Batched linearization of matching cost factors (Eqs. 2-8; Fig. 4 / P:224:
   inputs serialized into one block, one H2D, all factors processed in one
   fused launch, results serialized, one D2H).  Stateless: correspondences and
   Omega are recomputed at the given linearization points every call (P:208,
   P:313).
   factors, poses: host arrays (poses: num_poses x 12).  out: num_factors
   records in `mem`.  corr_dump (optional, DEVICE, int64 [sum_f N_f][L_f] packed
   per factor in factor order, L_f = levels of the factor's map): the packed key
   of each correspondence, -1 none, -2 discarded by validation.
   Errors: GVOX_ERR_INVALID with the factor index for an out-of-range cloud /
   map / pose index; non-finite poses. */
gvox_status gvox_linearize_batch(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                 int64_t num_clouds, const gvox_map* const* maps, int64_t num_maps,
                                 const gvox_factor* factors, int64_t num_factors,
                                 const double* poses, int64_t num_poses, gvox_linear_factor* out,
                                 int mem, int64_t* corr_dump);

/* Same, compact target-block records (for sharded runs and the NCCL gather). */
gvox_status gvox_linearize_batch_accum(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                       int64_t num_clouds, const gvox_map* const* maps,
                                       int64_t num_maps, const gvox_factor* factors,
                                       int64_t num_factors, const double* poses, int64_t num_poses,
                                       gvox_factor_accum* out, int mem);

/* Screened batch (P:391 factor creation followed by the Fig. 4 / P:224 batched
   linearization, with the screening decision kept on the device):
   candidates[p] (host, num_candidates) is a factor for every candidate pair;
   selected (DEVICE, uint8 [num_candidates]) is e.g. gvox_overlap_select's
   output with mem = GVOX_DEVICE.  The selected candidates, in candidate order,
   are compacted ON THE DEVICE and linearized exactly as
   gvox_linearize_batch_accum would linearize that list (the same records
   bitwise: a factor's result depends on the factor alone): out[k] (DEVICE,
   capacity num_candidates) is the k-th selected candidate's record,
   k < *num_selected (host out).  selected_host (optional, HOST,
   num_candidates bytes) receives a copy of the decisions.  One H2D (the
   candidate table), one 16-byte D2H before the launch (the selected and tile
   counts, and the kernel class of the SELECTED candidates -- OR of their
   hash-level / non-FAST / validation bits and their maximum level count,
   reduced on the device during the compaction -- plus the optional decision
   copy); returns with the linearization enqueued on ctx's stream.  The kernel
   variant (FAST all-dense / generic) is therefore the one
   gvox_linearize_batch_accum picks for the selected list: an unselected
   candidate with a hash level or a non-dyadic map does not change it.  Tile
   partials are sized for every candidate.  Errors as
   gvox_linearize_batch_accum. */
gvox_status gvox_linearize_batch_accum_select(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                              int64_t num_clouds, const gvox_map* const* maps,
                                              int64_t num_maps, const gvox_factor* candidates,
                                              int64_t num_candidates, const uint8_t* selected,
                                              const double* poses, int64_t num_poses,
                                              gvox_factor_accum* out, int64_t* num_selected,
                                              uint8_t* selected_host);

/* Expand compact records (DEVICE, e.g. after an all-gather) into full records:
   accum[k] belongs to factors[k]; poses as in gvox_linearize_batch (host).
   out in `mem`. */
gvox_status gvox_expand(gvox_ctx* ctx, const gvox_factor* factors, int64_t num_factors,
                        const double* poses, int64_t num_poses, const gvox_factor_accum* accum,
                        gvox_linear_factor* out, int mem);

/* ------------------------------------------------------ on-device registration */

/* Iterated re-linearization with a pose update on the device, no host round
   trip between iterations (the paper re-evaluates every
   matching cost factor in each optimization iteration, with Omega fixed
   at the linearization point).

   Every factor's pose_i is a VARIABLE pose; every pose_j is FIXED.  A pose may
   not be both (that couples poses into a joint system: GVOX_ERR_INVALID), and
   pose_i != pose_j.  The variable poses are therefore independent problems,
   solved together in one batch.  For a variable pose v, iteration k:
     1. linearize all factors with pose_i = v at (T_v^k, T_j) (Eqs. 2-8);
     2. H = sum_f H_ii(f), b = sum_f b_i(f), e_k = sum_f error(f), summed in
        ascending factor order;
     3. solve (H + lambda I) delta = -b by Cholesky (fp64); if the matrix is not
        positive definite the pose stops with GVOX_REG_SINGULAR, unchanged;
     4. T_v^(k+1) = T_v^k Exp(delta) (right perturbation, rotation-first
        delta = [w; rho], full SE(3) exponential);
     5. stop with GVOX_REG_CONVERGED when |w| <= eps_rot and |rho| <= eps_trans,
        or with GVOX_REG_MAX_ITER after max_iterations linearizations.
   The returned pose is the one after the last step, error_final the error at
   the last linearization.  One loop iteration = linearize + per-factor reduce
   + solve/update kernels, run as the body of a CUDA graph WHILE node whose
   condition the solve kernel sets (any pose still active): one graph launch
   per call, one H2D and (host outputs) one D2H.
   Converged poses stay frozen while others iterate. */
typedef struct gvox_register_params {
  int32_t max_iterations; /* linearizations per variable pose, in [1, 1000] */
  int32_t reserved;       /* 0 */
  double lambda;          /* >= 0; 0 = Gauss-Newton */
  double eps_rot;         /* >= 0 [rad] */
  double eps_trans;       /* >= 0 [m] */
} gvox_register_params;

enum {
  GVOX_REG_FIXED = 0,     /* not a variable pose (no factor has it as pose_i) */
  GVOX_REG_MAX_ITER = 1,
  GVOX_REG_CONVERGED = 2,
  GVOX_REG_SINGULAR = 3
};

typedef struct gvox_register_result {
  int32_t status;        /* GVOX_REG_* */
  int32_t iterations;    /* linearizations performed */
  int32_t inliers;       /* correspondences (all factors, all levels) at the last linearization */
  int32_t reserved;
  double error_initial;  /* e at the first linearization */
  double error_final;    /* e at the last linearization */
  double last_step[6];   /* the last delta applied (zeros when singular) */
} gvox_register_result;

/* factors, poses, params: host.  poses_out [num_poses x 12] (fixed poses copied
   unchanged), results [num_poses] (indexed by pose) and error_history
   (optional, [max_iterations x num_poses], e_k of pose v at [k * num_poses + v],
   0 after the pose stopped) live in `mem`. */
gvox_status gvox_register_batch(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                int64_t num_clouds, const gvox_map* const* maps, int64_t num_maps,
                                const gvox_factor* factors, int64_t num_factors,
                                const double* poses, int64_t num_poses,
                                const gvox_register_params* params, double* poses_out,
                                gvox_register_result* results, double* error_history, int mem);

/* ---------------------------------------------------------- global system */

/* One Gauss-Newton step of a whole factor graph of matching cost factors
   (global mapping; the solver the paper runs on the CPU, P:814;
   SURVEY §8(f) NEXT-4).  Poses with fixed[v] != 0 are constants (at least one
   is needed to remove the 6-dof gauge freedom, unless lambda > 0); the others
   are the variables, ordered by pose index.  With every factor's full blocks
   (H_ii, H_ij, H_jj, b_i, b_j; from its compact record `accum` and the poses,
   as gvox_expand) scattered onto its variable poses,
       H = sum_f scatter(H_f) + lambda I,   b = sum_f scatter(b_f),
   the step solves H delta = -b by block-Jacobi preconditioned conjugate
   gradients in fp64 until |r| <= tol |b| or max_iterations (the PCG loop runs
   on the device as a CUDA-graph WHILE node).  delta [num_poses x 6]
   (rotation-first, right perturbation: T_v <- T_v Exp(delta_v); 0 for fixed
   poses).  Every block and right-hand-side entry is summed in ascending
   factor order: results are bitwise reproducible.
   factors, poses, fixed, params: host.  accum [num_factors] and delta live in
   `mem`; H_dense [(6V)^2] and b_dense [6V] (optional, HOST, row-major, V =
   variables) receive the assembled system for inspection.
   Errors: GVOX_ERR_INVALID for bad indices / sizes, no fixed pose with
   lambda = 0, or a diagonal block that is not positive definite. */
typedef struct gvox_global_params {
  int32_t max_iterations; /* PCG iterations, >= 1 */
  int32_t reserved;
  double tol;             /* relative residual, >= 0 */
  double lambda;          /* >= 0, added to the diagonal */
} gvox_global_params;

typedef struct gvox_global_result {
  int32_t iterations;     /* PCG iterations run */
  int32_t converged;      /* |r| <= tol |b| */
  int32_t num_variables;
  int32_t num_blocks;     /* stored 6x6 blocks (both triangles) */
  double residual_initial; /* |b| */
  double residual_final;   /* |r| (recurrence) */
} gvox_global_result;

gvox_status gvox_solve_global(gvox_ctx* ctx, const gvox_factor* factors, int64_t num_factors,
                              const gvox_factor_accum* accum, const double* poses,
                              int64_t num_poses, const uint8_t* fixed,
                              const gvox_global_params* params, double* delta, double* H_dense,
                              double* b_dense, gvox_global_result* result, int mem);

/* Gauss-Newton optimisation of the whole graph (the global mapping loop,
   P:391, with every factor re-linearized at every iteration).  Each
   iteration: gvox_linearize_batch_accum at the current poses (device
   records), gvox_solve_global (params' PCG settings), T_v <- T_v Exp(delta_v)
   on the device; stop when max_v |w_v| <= eps_rot and max_v |rho_v| <=
   eps_trans, or after max_iterations.  error_history (optional, HOST,
   [max_iterations]) receives the total error at each linearization.
   clouds, maps, factors, poses, fixed, params: as in gvox_linearize_batch /
   gvox_solve_global (host); poses_out [num_poses x 12] in `mem`. */
typedef struct gvox_optimize_params {
  int32_t max_iterations;      /* Gauss-Newton iterations, >= 1 */
  int32_t pcg_max_iterations;  /* per solve, >= 1 */
  double pcg_tol;
  double lambda;
  double eps_rot;              /* rad */
  double eps_trans;            /* m */
} gvox_optimize_params;

typedef struct gvox_optimize_result {
  int32_t iterations;          /* linearizations performed */
  int32_t converged;
  int32_t pcg_iterations;      /* summed over the solves */
  int32_t reserved;
  double error_initial;        /* total error at the first linearization */
  double error_final;          /* ... at the last one */
  double last_step_rot;        /* max |w| of the last step */
  double last_step_trans;      /* max |rho| of the last step */
} gvox_optimize_result;

gvox_status gvox_optimize_global(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                 int64_t num_clouds, const gvox_map* const* maps, int64_t num_maps,
                                 const gvox_factor* factors, int64_t num_factors,
                                 const double* poses, int64_t num_poses, const uint8_t* fixed,
                                 const gvox_optimize_params* params, double* poses_out,
                                 double* error_history, gvox_optimize_result* result, int mem);

/* ------------------------------------------------------------- utilities */

const char* gvox_status_string(gvox_status s);
const char* gvox_last_error(void);
/* Kernel launches issued by this thread since the last reset (evidence for
   bench.py's gpu_launches). */
int64_t gvox_launch_count(int reset);
/* The k_linearize instantiation this thread launched last (introspection for
   tests and tools; 0 before any linearization): GVOX_LINVAR_FAST (the
   specialised 3-level dyadic kernel), GVOX_LINVAR_DENSE (all levels dense
   grids), GVOX_LINVAR_VALID (P:197 visibility test compiled in) | the kernel's
   level capacity << 8.  The records do not depend on it (the variants are
   bitwise equal, tested); only the speed does. */
#define GVOX_LINVAR_FAST 1
#define GVOX_LINVAR_DENSE 2
#define GVOX_LINVAR_VALID 4
int32_t gvox_last_linearize_variant(void);
const char* gvox_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GVOX_H_ */
