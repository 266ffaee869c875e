// gvox_internal.h -- device-side data layout shared by the runtime
// (gvox_runtime.cu) and the kernels (k_*.cu).  Not part of the ABI.
//
// HBM layout:
//  * cloud: 48 B/point in chunks of 32 points (1536 B): each chunk holds the
//    three float4 planes of its 32 points back to back,
//      A[k] = {mu.x, mu.y, mu.z, C.xx}
//      B[k] = {C.xy, C.xz, C.yy, C.yz}
//      N[k] = {C.zz, n.x, n.y, n.z}
//    at float4 offset pt_off(k) from A, B = A + 32, N = A + 64 (so one pointer
//    plus immediates reaches all three planes of a warp's 32 points); the
//    overlap kernel streams only A (512 B runs, 16 B/point); linearize all 3.
//  * map level: open-addressing hash of 16 B slots {u64 packed key, i32 voxel
//    index, pad} (capacity 2^k >= 2V, EMPTY key = ~0) + compact voxel records
//    of 48 B: {off.x, off.y, off.z, C.xx}, {C.xy, C.yy, C.xz, C.yz},
//    {C.zz, count (int bits), 0, 0}; `off` = voxel mean minus voxel centre in
//    fp32 (the residual is formed as fp32(centre - q64) + off, reading Q12);
//    + the packed key per voxel (u64) for export.
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/gvox.h"

namespace gvox {

constexpr uint64_t kEmptyKey = ~0ull;
constexpr int kKeyBits = 21;
constexpr int32_t kKeyHalf = 1 << 20;

constexpr int kChunk = 32;  // points per layout chunk (also the culling box granularity)
// float4 offset of point k's A record from the cloud's A pointer (B, N: + 32, + 64)
__host__ __device__ __forceinline__ int64_t pt_off(int64_t k) { return (k >> 5) * 96 + (k & 31); }
// float4 slots a cloud of n points occupies
__host__ __device__ __forceinline__ int64_t pt_slots(int64_t n) { return ((n + 31) >> 5) * 96; }

struct CloudDev {
  const float4* A;
  const float4* B;
  const float4* N;
  // bounding box of every 32 consecutive points (a warp's worth):
  // [chunk] = {min.x, min.y, min.z, max.x, max.y, max.z}, ceil(n / 32) chunks
  const float* chunk_box;
  int64_t n;
  int32_t has_normals;
  int32_t pad;
};

// One level of a map.  Voxel lookup uses either
//  * a DENSE index grid over the level's key bounding box (int32 voxel index
//    or -1 per cell; chosen before the build when the box has at most
//    kDenseBuildRatio cells per point): one predicated load, no probing; or
//  * the open-addressing HASH table (sparse / very large extents).
struct __align__(16) MapLevelDev {
  // dense-grid fields first, 16 B aligned: two vector loads per lookup
  int32_t x0, y0, z0;       // dense: key of cell (0, 0, 0)
  uint32_t dx;              // dense: box size in cells (each < 2^30, product < 2^31)
  uint32_t dy, dz;
  uint32_t syz;             // dy * dz (x stride)
  int32_t dense;            // 1 = dense grid
  const int32_t* grid;      // dense: [dx * dy * dz], x-major; nullptr for hash
  const float4* vox;        // [3 * nvox]
  const ulonglong2* slots;  // hash: [mask + 1] {key, idx}
  uint64_t mask;            // hash capacity - 1
  double r;      // r0 * 2^l
  double inv_r;  // 1 / r (used only when dyadic)
  int64_t nvox;
  int32_t shift;            // 64 - log2(capacity)
  int32_t pad;
};

// linearize tile plan: tiles of 256 * ppt points of one factor, ppt = the
// largest power of two <= GVOX_TILE_MAX_PPT with n >= 256 * MIN_TILES * ppt
// (a function of the factor alone: batch == serial bit for bit)
#ifndef GVOX_TILE_MAX_PPT
#define GVOX_TILE_MAX_PPT 128
#endif
#ifndef GVOX_TILE_MIN_TILES
#define GVOX_TILE_MIN_TILES 2
#endif
// factors below GVOX_TILE_SMALL_N points (odometry frames, ~20k) are cut into
// at least GVOX_TILE_MIN_TILES_SMALL tiles: their batches are small, so the
// tiles must spread over the SMs (still a function of the factor alone)
#ifndef GVOX_TILE_SMALL_N
#define GVOX_TILE_SMALL_N 32768
#endif
#ifndef GVOX_TILE_MIN_TILES_SMALL
#define GVOX_TILE_MIN_TILES_SMALL 16
#endif

#ifndef GVOX_DENSE_RATIO
#define GVOX_DENSE_RATIO 2048
#endif
constexpr int kDenseBuildRatio = GVOX_DENSE_RATIO;  // max cells per POINT for a dense grid level

struct MapDev {
  int32_t levels;
  int32_t dyadic;  // r0 is a power of two: floor(q * inv_r0) == floor(q / r0)
  double r0;
  double inv_r0;
  // conservative box of every voxel of every level: the source cloud's box
  // grown by the coarsest resolution (a point q can only hit a voxel whose
  // cell contains a map point p, so |q - p| < r_l per axis).  Empty map: lo > hi.
  float box_lo[4], box_hi[4];
  MapLevelDev lv[GVOX_MAX_LEVELS];
};

// Per-tile partial of the linearize kernel (doubles; counts stored exactly).
constexpr int kNumTerms = 28;
constexpr int kPartialStride = 40;  // 28 terms, 8 inliers, invisible, degenerate, 2 pad

// Fibonacci (multiplicative) hashing: the TOP log2(capacity) bits of
// key * 2^64/phi, i.e. shift = 64 - log2(capacity).  (The low bits of the
// product depend only on the low bits of the key, which would ignore kx.)
// The probe sequence is linear.
__host__ __device__ inline uint64_t hash_slot(uint64_t key, int shift) {
  return (key * 0x9E3779B97F4A7C15ull) >> shift;
}

inline int shift_for_capacity(uint64_t cap) {  // cap = 2^k, k >= 1
  int k = 0;
  while ((1ull << k) < cap) ++k;
  return 64 - k;
}

__host__ __device__ inline uint64_t pack_key(int32_t kx, int32_t ky, int32_t kz) {
  return ((uint64_t)(uint32_t)(kx + kKeyHalf) << 42) | ((uint64_t)(uint32_t)(ky + kKeyHalf) << 21) |
         (uint64_t)(uint32_t)(kz + kKeyHalf);
}

__host__ __device__ inline bool key_in_range(int32_t k) { return k >= -kKeyHalf && k < kKeyHalf; }

// ---------------------------------------------------------------- launchers
// (defined in k_*.cu; all asynchronous on `stream`)

// cloud: pack user arrays into the planar layout and reduce per-cloud stats
// (8 int32): [0] |= 1 on non-finite input, [1] = max |C_ij| (float bits),
// [2..4] = min mu, [5..7] = max mu (order-preserving int encoding of floats;
// initialise [2..4] to INT_MAX and [5..7] to INT_MIN).
void launch_cloud_pack(const float* mu, const float* cov, const float* nrm, int64_t n, float4* P,
                       float* chunk_box, int32_t* stats, cudaStream_t stream);
// the same for every cloud of a batch in one launch (count <= 65535)
struct PackSeg {
  const float* mu;
  const float* cov;
  const float* nrm;  // or nullptr
  int64_t n;
  float4* P;
  float* chunk_box;
  int32_t* stats;    // 8 int32 as above
};
void launch_cloud_pack_batch(const PackSeg* segs_dev, int64_t count, int64_t max_n,
                             cudaStream_t stream);

__host__ __device__ inline int32_t float_to_ordered(float f) {
#ifdef __CUDA_ARCH__
  int32_t i = __float_as_int(f);
#else
  int32_t i;
  memcpy(&i, &f, 4);
#endif
  return i < 0 ? i ^ 0x7FFFFFFF : i;
}
__host__ __device__ inline float ordered_to_float(int32_t i) {
  int32_t j = i < 0 ? i ^ 0x7FFFFFFF : i;
#ifdef __CUDA_ARCH__
  return __int_as_float(j);
#else
  float f;
  memcpy(&f, &j, 4);
  return f;
#endif
}

// voxelmap build.  A level is DENSE (an int32 index grid over its key box,
// decided before the build from the cloud's bounding box) or HASH (sparse
// extents).  Phase 1 assigns each new voxel a compact index: dense levels CAS
// the final grid cell directly; hash levels insert into a temporary table and
// record per (point, level) the slot of their key.
struct LevelBox {
  int32_t x0, y0, z0;
  uint32_t dx, dy, dz, syz;
  int32_t dense;
  int32_t* grid;            // dense: the map's final grid (0xFF-filled), else nullptr
};
struct BuildSeg {
  const float4* A;          // cloud means (+C.xx)
  int64_t n;                // points
  int64_t pl_offset;        // this cloud's first point in the level-major (level, point) slots
  int64_t pl_stride;        // slots per level (the chunk's points): coalesced per level
  ulonglong2* tmp_slots[GVOX_MAX_LEVELS];  // hash levels: temp tables (capacity tmp_mask+1)
  uint64_t tmp_mask;
  int32_t tmp_shift;
  int32_t lift;  // 1: only level 0 accumulated from the points, coarser levels lifted (k_build_lift)
  uint64_t* keys_by_idx[GVOX_MAX_LEVELS];  // [n] workspace: key of voxel idx
  int32_t* counter;         // [levels] voxel counts (atomic)
  // sync-free builds (acc sized by upper bounds before the insert): the
  // thread that creates voxel idx of level l zeroes its 10 accumulators at
  // acc + (acc_offset[l] + idx) * 10; nullptr: acc is zero-filled instead
  unsigned long long* acc;
  int64_t acc_offset[GVOX_MAX_LEVELS];
  LevelBox box[GVOX_MAX_LEVELS];
  // hash levels: phase 1 records, per (point, level), the temp-table SLOT of its
  // key; phase 2 reads the voxel index from that slot (all assigned by then).
};
void launch_build_insert(const BuildSeg* segs_dev, int64_t num_segs, int64_t max_seg_points,
                         int levels, double r0, int dyadic, int32_t* pslot, int32_t* err,
                         cudaStream_t stream);

// phase 2: fixed-point accumulation of (sum offsets, sum cov, count) per voxel.
struct AccumSeg {
  const float4* A;
  const float4* B;
  const float4* N;
  int64_t n;
  int64_t pl_offset;
  int64_t pl_stride;
  int64_t acc_offset[GVOX_MAX_LEVELS];  // first voxel of (seg, level) in acc[]
  double mu_scale[GVOX_MAX_LEVELS];     // offset scale: 2^F / r_l, or (lifted builds) 2^F / r_(L-1) for every l
  double cov_scale;                     // 2^(F - e_c), 2^e_c >= max |C_ij| of the cloud
};
void launch_build_accum(const BuildSeg* bsegs_dev, const AccumSeg* segs_dev, int64_t num_segs,
                        int64_t max_seg_points, int levels, double r0, int dyadic,
                        const int32_t* pslot, unsigned long long* acc, cudaStream_t stream);

// phase 2b: coarser levels from finer ones (nested voxels; see k_build.cu)
void launch_build_lift(const BuildSeg* bsegs_dev, const AccumSeg* segs_dev, int64_t num_segs,
                       int levels, const int64_t* max_level_voxels, double r0,
                       unsigned long long* acc, cudaStream_t stream);

// phase 3: per voxel, finalize the record and insert into the final table.
struct FinalSeg {
  int64_t acc_offset;       // first voxel in acc[] / keys
  const int32_t* nvox;      // device: the level's voxel count (the insert's counter)
  int32_t* nvox_out;        // device: the map's copy of it (written by the finalize)
  const uint64_t* keys_by_idx;
  double r;
  double mu_scale;
  double cov_scale;
  ulonglong2* slots;        // final table
  uint64_t mask;
  int32_t shift;
  int32_t dense;
  int32_t* grid;            // dense index grid (or nullptr)
  int32_t x0, y0, z0;
  uint32_t dx, dy, dz;
  float4* vox;              // [3 * nvox]
  uint64_t* keys_out;       // [nvox]
};
void launch_build_finalize(const FinalSeg* segs_dev, int64_t num_segs, int64_t max_seg_voxels,
                           const unsigned long long* acc, cudaStream_t stream);

void launch_fill_u64(uint64_t* p, uint64_t value, int64_t count, cudaStream_t stream);
// H2D of a small pinned block by an SM kernel (no copy engine)
void launch_h2d_copy(void* dst, const void* pinned_src, int64_t bytes, cudaStream_t stream);
// up to 4 segments in ONE launch: copy pinned src -> dst, or zero-fill dst
// when src is NULL (a call's input blocks and the zeroing of its counters)
struct H2DSeg {
  void* dst;
  const void* src;
  int64_t bytes;
};
void launch_h2d_segments(const H2DSeg* segs, int n, cudaStream_t stream);
// blocks of at most this many bytes go up inside the launch's parameters (the
// pinned source is free again as soon as the launch is enqueued)
int64_t h2d_param_max();

// Recycling of dense index grids (gvox_runtime.cu GridArena): a dense level's
// only non-empty cells are its voxels' cells, so writing -1 back into exactly
// those cells returns the grid to the all-empty state a build expects -- V
// scattered stores instead of a fill of the whole box.
struct ResetSeg {
  const uint64_t* keys;  // the level's packed voxel keys [nvox]
  int32_t* grid;
  const int32_t* nvox;   // device: the level's voxel count (nullptr: not a dense level)
  int32_t x0, y0, z0;
  uint32_t dy, dz;
};
void launch_grid_reset(const ResetSeg* segs_dev, int64_t num_segs, int64_t max_seg_voxels,
                       cudaStream_t stream);

// lookup
void launch_lookup(const MapDev* map, int level, const double* q, int64_t n, int64_t* out,
                   cudaStream_t stream);

// overlap
struct PairDev {
  int32_t src, tgt, pi, pj;
};
void launch_overlap(const CloudDev* const* clouds, const MapDev* const* maps, const PairDev* pairs,
                    const int32_t* tile_start, int64_t num_pairs, int64_t num_tiles, int tile_pts,
                    const double* poses, int level, int32_t* tile_pair, int32_t* counts,
                    bool all_dense, cudaStream_t stream);

void launch_overlap_select(const CloudDev* const* clouds, const MapDev* const* maps,
                           const PairDev* pairs, int64_t num_pairs, const double* poses, int level,
                           int32_t num, int32_t den, uint8_t* selected, bool all_dense,
                           bool all_dyadic, cudaStream_t stream);

// union overlap (P:280 keyframe insertion): query q = source cloud at pose pi
// against members[first, first + count) = {target map, pose_j}
struct UnionQueryDev {
  int32_t src, pi, first, count;
};
struct UnionMemberDev {
  int32_t tgt, pj;
};
// tiles of tile_pts <= 256 * 32 points
void launch_overlap_union(const CloudDev* const* clouds, const MapDev* const* maps,
                          const UnionQueryDev* queries, const UnionMemberDev* members,
                          const int32_t* tile_start, const int32_t* tile_query, int64_t num_tiles,
                          int tile_pts, const double* poses, int level, int32_t* counts,
                          cudaStream_t stream);

// preprocessing (k_knn.cu): per cloud, a uniform cell grid over its bounding
// box; the cloud's points are [first, first + n) of the batch arrays and its
// cells [cell0, cell0 + dim0 * dim1 * dim2) of the global cell arrays
struct KnnCloudDev {
  int64_t first, n;
  double lo[3];
  double s, inv_s;
  int32_t dim[3];
  int32_t cell0;
};
void launch_knn_bbox(const float* pts, const KnnCloudDev* clouds, const int32_t* tile_start,
                     const int32_t* tile_cloud, int64_t num_tiles, int tile_pts, int32_t* box,
                     int32_t* bad, cudaStream_t stream);
void launch_knn_count(const float* pts, const KnnCloudDev* clouds, const int32_t* tile_start,
                      const int32_t* tile_cloud, int64_t num_tiles, int tile_pts, int32_t* cell_of,
                      int32_t* count, cudaStream_t stream);
void launch_exclusive_scan(const int32_t* in, int64_t n, int32_t* out, int32_t* scratch,
                           cudaStream_t stream);
void launch_knn_scatter(const float* pts, const KnnCloudDev* clouds, const int32_t* tile_start,
                        const int32_t* tile_cloud, int64_t num_tiles, int tile_pts,
                        const int32_t* cell_of, const int32_t* cell_start, int32_t* fill,
                        float4* sorted, cudaStream_t stream);
void launch_knn_query(const KnnCloudDev* clouds, const int32_t* tile_start, const int32_t* tile_cloud,
                      int64_t num_tiles, int tile_pts, const float4* sorted,
                      const int32_t* cell_start, int k, int32_t* out, cudaStream_t stream);
void launch_covariance(const float* pts, const KnnCloudDev* clouds, const int32_t* tile_start,
                       const int32_t* tile_cloud, int64_t num_tiles, int tile_pts, const int32_t* nbr,
                       int k, float* cov, float* nrm, cudaStream_t stream);

// linearize
struct FactorDev {
  int32_t src, tgt, pi, pj;
  uint32_t flags;
  int32_t tile_pts;     // points per tile of this factor (a function of its own size
                        // only, so results do not depend on the rest of the batch)
  int64_t corr_offset;  // first (point, level) record in corr_dump
};
void launch_linearize(const CloudDev* const* clouds, const MapDev* const* maps,
                      const FactorDev* factors, const int32_t* tile_start, int64_t num_factors,
                      int64_t num_tiles, int tile_pts, int max_levels, const double* poses,
                      double* partials, int32_t* tile_factor, int64_t* corr_dump,
                      bool all_dense, bool fast, bool validate, cudaStream_t stream,
                      const int32_t* exec_order = nullptr /* [num_tiles] block -> tile */);
// execution order of a screened batch's tiles grouped by target map (device
// counting sort; hist: num_maps int32 workspace)
void launch_exec_order_by_target(const FactorDev* fc, const int32_t* tsc, int64_t S,
                                 int64_t num_maps, int32_t* hist, int32_t* exec,
                                 cudaStream_t stream);
// reduce tile partials per factor in fixed order; write full or compact records.
void launch_reduce(const FactorDev* factors, const int32_t* tile_start, int64_t num_factors,
                   const double* poses, const double* partials, gvox_linear_factor* out_full,
                   gvox_factor_accum* out_accum, cudaStream_t stream);
void launch_expand(const FactorDev* factors, int64_t num_factors, const double* poses,
                   const gvox_factor_accum* accum, gvox_linear_factor* out, cudaStream_t stream);

// on-device registration (gvox_register_batch): one problem per variable pose,
// its factors at reg_factors[f0, f1) in ascending factor order.
struct RegProblem {
  int32_t pose, f0, f1, pad;
};
struct RegControl {
  int32_t iter;          // loop iterations completed
  int32_t max_iter;
  int32_t any_active;    // per-iteration count (reset by the last block)
  uint32_t blocks_done;  // per-iteration block ticket (reset by the last block)
  double lambda, eps_rot, eps_trans;
};
void launch_gn_step(const RegProblem* problems, int32_t num_problems, const int32_t* reg_factors,
                    const FactorDev* factors, const gvox_factor_accum* accum, double* poses,
                    gvox_register_result* results, int32_t* active, RegControl* ctrl,
                    double* history, int64_t num_poses, cudaGraphConditionalHandle cond,
                    cudaStream_t stream);

// global system (k_global.cu): BSR assembly + block-Jacobi PCG
struct PcgState {
  double rz, r0, res;
  int32_t iter, done;
};
void launch_assemble(const gvox_linear_factor* rec, const int32_t* contrib_start,
                     const int32_t* contrib, int64_t num_blocks, const uint8_t* is_diag,
                     double lambda, double* blocks, const int32_t* g_start, const int32_t* g_list,
                     int64_t num_vars, double* rhs, const int32_t* diag_block, double* minv,
                     int32_t* bad, cudaStream_t stream);
void launch_pcg_init(const double* rhs, const double* minv, int64_t num_vars, double* x, double* r,
                     double* z, double* p, PcgState* st, cudaStream_t stream);
void launch_pcg_iteration(const double* blocks, const int32_t* row_start, const int32_t* col,
                          int64_t num_vars, const double* minv, double* x, double* r, double* z,
                          double* p, double* q, double* pq_part, PcgState* st, int32_t max_iter,
                          double tol, cudaGraphConditionalHandle cond, cudaStream_t stream);
bool launch_pcg_cluster(const double* blocks, const int32_t* row_start, const int32_t* col,
                        int64_t num_vars, int64_t num_blocks, const double* minv, const double* rhs,
                        double* x, double* r, double* z, double* p, double* q, PcgState* st,
                        int32_t max_iter, double tol, cudaStream_t stream);
void launch_pcg_persistent(const double* blocks, const int32_t* row_start, const int32_t* col,
                           int64_t num_vars, const double* minv, const double* rhs, double* x,
                           double* r, double* z, double* p, double* q, double* part_a,
                           double* part_b, PcgState* st, int32_t max_iter, double tol,
                           const int32_t* chunk_row, const int32_t* chunk_b0,
                           const int32_t* row_chunk, int64_t num_chunks, double* qpart,
                           double* part_c, cudaStream_t stream);
void launch_scatter_delta(const double* x, const int32_t* var_of_pose, int64_t num_poses,
                          double* delta, cudaStream_t stream);

void launch_apply_delta(double* poses, const double* delta, int64_t num_poses, double* out_max,
                        cudaStream_t stream);
void launch_sum_error(const gvox_factor_accum* acc, int64_t n, double* out, cudaStream_t stream);

// tile -> owning item (factor or pair) table from the tile prefix sums
void launch_tile_map(const int32_t* tile_start, int64_t num_items, int32_t* tile_owner,
                     cudaStream_t stream);
// compact the selected candidates (device plan of gvox_linearize_batch_accum_select)
// counts (4 int32): {selected, their tiles, OR of their class bits, max of their levels};
// cls: per-candidate kernel-class byte (gvox_runtime.cu kCls*, levels << 4)
void launch_select_plan(const uint8_t* selected, const int32_t* ntiles, const uint8_t* cls,
                        const FactorDev* factors, int64_t num_cand, FactorDev* factors_c,
                        int32_t* tile_start_c, int32_t* counts,
                        int2* block_tot /* ceil(num_cand / 1024) */, cudaStream_t stream);

void note_launch();
// the k_linearize instantiation just launched: GVOX_LINVAR_* bits | MAXL << 8
void note_linearize_variant(int32_t v);

}  // namespace gvox
