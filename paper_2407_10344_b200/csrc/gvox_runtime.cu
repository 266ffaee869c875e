// gvox_runtime.cu -- host runtime behind the C ABI of include/gvox.h:
// contexts, device-resident cloud and map handles, the batch serializer
// (P:224 / Fig.4: inputs serialized into ONE host block, ONE H2D, fused
// launches, ONE D2H), workspace management and error reporting.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include <chrono>
#include <cstdlib>

#include "gvox_internal.h"

using namespace gvox;

namespace {
// GVOX_DEBUG_TIMING=1: host-side phase timings of the map build on stderr
struct DebugClock {
  bool on = std::getenv("GVOX_DEBUG_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char* what) {
    if (!on) return;
    auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[gvox build] %-22s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};
}  // namespace

// ------------------------------------------------------------------ errors
namespace {
thread_local std::string g_last_error;
thread_local int64_t g_launches = 0;
thread_local int32_t g_lin_variant = 0;  // the last k_linearize instantiation (gvox_last_linearize_variant)

gvox_status fail(gvox_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

gvox_status cuda_fail(cudaError_t e, const char* where) {
  cudaGetLastError();  // clear sticky-free errors
  if (e == cudaErrorMemoryAllocation)
    return fail(GVOX_ERR_NOMEM, "%s: %s", where, cudaGetErrorString(e));
  return fail(GVOX_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(call)                                        \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

#define CK_LAUNCH(where)                                 \
  do {                                                   \
    cudaError_t e_ = cudaGetLastError();                 \
    if (e_ != cudaSuccess) return cuda_fail(e_, where);  \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  bool changed = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) {
      changed = cudaSetDevice(dev) == cudaSuccess;
    }
  }
  ~DeviceGuard() {
    if (changed) cudaSetDevice(prev);
  }
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

uint64_t pow2_at_least(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

bool finite_pose(const double* T) {
  for (int i = 0; i < 12; ++i)
    if (!std::isfinite(T[i])) return false;
  return true;
}

bool is_dyadic(double r) {
  int e;
  return std::frexp(r, &e) == 0.5;
}

// A device allocation shared by the handles carved out of it.  Stream-ordered:
// allocated from the device's default memory pool on the creating context's
// stream and returned to the pool on that stream when the last handle goes
// (handles must therefore be destroyed before that stream is).
// Recycled record arenas (small builds rebuild maps of about the same size
// every frame): a released arena is parked here instead of freed, and the next
// build on the SAME stream that needs at most that many bytes (and at least
// half) takes it -- stream order already puts the new build after everything
// that used it.  At most kRecPoolKeep are kept.
constexpr size_t kRecPoolKeep = 2;
struct RecPool {
  struct Entry {
    void* ptr;
    size_t bytes;
    cudaStream_t stream;
  };
  std::mutex mu;
  std::vector<Entry> free;
  int device = 0;
  static void release(const Entry& e, int device) {
    DeviceGuard g(device);
    if (cudaFreeAsync(e.ptr, e.stream) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(e.ptr);
    }
  }
  ~RecPool() {
    for (const Entry& e : free) release(e, device);
  }
};

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::shared_ptr<RecPool> pool;  // null: freed, not recycled
  ~DevBuf() {
    if (!ptr) return;
    if (pool) {
      std::lock_guard<std::mutex> lk(pool->mu);
      pool->free.push_back({ptr, bytes, stream});
      while (pool->free.size() > kRecPoolKeep) {
        RecPool::release(pool->free.front(), device);
        pool->free.erase(pool->free.begin());
      }
      return;
    }
    DeviceGuard g(device);
    if (cudaFreeAsync(ptr, stream) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(ptr);
    }
  }
};

gvox_status devbuf_alloc(size_t bytes, int device, cudaStream_t stream,
                         std::shared_ptr<DevBuf>* out,
                         const std::shared_ptr<RecPool>& pool = nullptr) {
  auto b = std::make_shared<DevBuf>();
  b->device = device;
  b->bytes = bytes;
  b->stream = stream;
  b->pool = pool;
  if (bytes && pool) {
    std::lock_guard<std::mutex> lk(pool->mu);
    size_t best = pool->free.size();
    for (size_t i = 0; i < pool->free.size(); ++i) {
      const RecPool::Entry& e = pool->free[i];
      if (e.stream == stream && e.bytes >= bytes && e.bytes <= 2 * bytes &&
          (best == pool->free.size() || e.bytes < pool->free[best].bytes))
        best = i;
    }
    if (best < pool->free.size()) {
      b->ptr = pool->free[best].ptr;
      b->bytes = pool->free[best].bytes;
      pool->free.erase(pool->free.begin() + best);
      *out = b;
      return GVOX_OK;
    }
  }
  if (bytes) {
    cudaError_t e = cudaMallocAsync(&b->ptr, bytes, stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  }
  *out = b;
  return GVOX_OK;
}

// Recycled dense index grids.  A build needs its grids all -1 (empty); a
// fresh arena gets a full fill, a recycled one is already clean: when the last
// map of a build goes, its GridArena writes -1 back into exactly the cells its
// voxels set (launch_grid_reset: V scattered stores instead of a fill of the
// whole key box -- at C5 ~6e7 cells instead of ~5e9) and parks the memory in
// its context's pool, from which the next build of about the same size takes
// it (stream-ordered after the reset by an event).  At most kGridPoolKeep
// arenas are kept; the pool outlives its context while arenas refer to it.
constexpr size_t kGridPoolKeep = 2;
struct GridPool {
  struct Entry {
    void* ptr;
    size_t bytes;
    cudaStream_t stream;
    cudaEvent_t ready;  // the reset that cleaned it has run
  };
  std::mutex mu;
  std::vector<Entry> free;
  std::vector<cudaEvent_t> spare;  // events of taken entries, reused (no create / destroy per build)
  int device = 0;
  static void release(const Entry& e, int device) {
    DeviceGuard g(device);
    if (cudaFreeAsync(e.ptr, e.stream) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(e.ptr);
    }
    cudaEventDestroy(e.ready);
  }
  ~GridPool() {
    for (const Entry& e : free) release(e, device);
    for (cudaEvent_t e : spare) cudaEventDestroy(e);
  }
};

struct GridArena {
  void* ptr = nullptr;
  size_t bytes = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::shared_ptr<GridPool> pool;  // null: freed, not recycled
  std::shared_ptr<DevBuf> rec;     // record arena: keys + reset table, alive until the reset ran
  const ResetSeg* reset = nullptr;
  int64_t nreset = 0, max_vox = 0;
  ~GridArena() {
    if (!ptr) return;
    DeviceGuard g(device);
    cudaEvent_t ev = nullptr;
    if (pool) {
      std::lock_guard<std::mutex> lk(pool->mu);
      if (!pool->spare.empty()) {
        ev = pool->spare.back();
        pool->spare.pop_back();
      }
    }
    if (pool && reset && (ev || cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess)) {
      launch_grid_reset(reset, nreset, max_vox, stream);
      if (cudaGetLastError() == cudaSuccess && cudaEventRecord(ev, stream) == cudaSuccess) {
        std::lock_guard<std::mutex> lk(pool->mu);
        pool->free.push_back({ptr, bytes, stream, ev});
        while (pool->free.size() > kGridPoolKeep) {  // the oldest goes back to the device pool
          GridPool::release(pool->free.front(), device);
          pool->free.erase(pool->free.begin());
        }
        return;  // (rec is released after this: its stream-ordered free follows the reset)
      }
      cudaGetLastError();
      cudaEventDestroy(ev);
    }
    if (cudaFreeAsync(ptr, stream) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(ptr);
    }
  }
};

// An all-empty grid arena of >= bytes: a recycled one (no fill needed, *fresh
// = false) of at most twice the size, else a new allocation (*fresh = true:
// the caller fills it with -1).
gvox_status grid_arena_take(const std::shared_ptr<GridPool>& pool, size_t bytes, int device,
                            cudaStream_t stream, std::shared_ptr<GridArena>* out, bool* fresh) {
  auto a = std::make_shared<GridArena>();
  a->device = device;
  a->stream = stream;
  a->bytes = bytes;
  *fresh = true;
  if (!bytes) {
    *out = a;
    *fresh = false;
    return GVOX_OK;
  }
  {
    std::lock_guard<std::mutex> lk(pool->mu);
    size_t best = pool->free.size();
    for (size_t i = 0; i < pool->free.size(); ++i) {
      const size_t b = pool->free[i].bytes;
      if (b >= bytes && b <= 2 * bytes && (best == pool->free.size() || b < pool->free[best].bytes))
        best = i;
    }
    if (best < pool->free.size()) {
      const GridPool::Entry e = pool->free[best];
      pool->free.erase(pool->free.begin() + best);
      if (e.stream != stream) CK(cudaStreamWaitEvent(stream, e.ready, 0));  // (same stream: ordered)
      pool->spare.push_back(e.ready);
      a->ptr = e.ptr;
      a->bytes = e.bytes;
      *fresh = false;
    }
  }
  if (*fresh) {
    cudaError_t e = cudaMallocAsync(&a->ptr, bytes, stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync (grid arena)");
  }
  a->pool = pool;
  *out = a;
  return GVOX_OK;
}

}  // namespace

namespace gvox {
void note_launch() { ++g_launches; }
void note_linearize_variant(int32_t v) { g_lin_variant = v; }
}  // namespace gvox

// ------------------------------------------------------------------ handles
struct gvox_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  // grow-only device workspaces
  void* ws[3] = {nullptr, nullptr, nullptr};
  size_t ws_bytes[3] = {0, 0, 0};
  // pinned host staging of the calls' single H2D input blocks: a ring of
  // slots, so a call only waits when the copy out of the slot it reuses (four
  // calls back) has not landed -- consecutive calls do not serialise the host
  // with the stream
  static constexpr int kPinSlots = 4;
  struct PinSlot {
    void* ptr = nullptr;
    size_t bytes = 0;
    cudaEvent_t done = nullptr;  // the last H2D out of this slot has completed
    bool pending = false;
  };
  PinSlot pin_ring[kPinSlots];
  int pin_slot = 0;
  // optional device-side kernel timing (gvox_ctx_enable_timing)
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_open[GVOX_TIMER_COUNT];
  double timer_ms[GVOX_TIMER_COUNT] = {};
  int64_t timer_launches[GVOX_TIMER_COUNT] = {};
  // gvox_register_batch: capture stream for the loop graph, pinned D2H staging
  cudaStream_t cap_stream = nullptr;
  void* pin_out = nullptr;
  size_t pin_out_bytes = 0;
  int32_t* pin_counts = nullptr;  // pinned {S, T} of gvox_linearize_batch_accum_select
  uint64_t dense_budget = 16ull << 30;  // bytes of dense index grids per build chunk
  std::shared_ptr<GridPool> grid_pool = std::make_shared<GridPool>();
  std::shared_ptr<RecPool> rec_pool = std::make_shared<RecPool>();  // record arenas of small builds
  // pinned staging of the build's two descriptor uploads (pageable copies
  // would wait for the stream to drain before they start)
  void* pin_b[2] = {nullptr, nullptr};
  size_t pin_b_bytes[2] = {0, 0};
  cudaEvent_t pin_b_done[2] = {nullptr, nullptr};
};

struct gvox_cloud {
  std::shared_ptr<DevBuf> buf;
  CloudDev desc{};       // host copy
  CloudDev* dev = nullptr;  // device copy of desc
  int64_t n = 0;
  float cmax = 0.f;      // max |C_ij| (fixed-point scale of the voxel build)
  float lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};  // bounding box of the means (n > 0)
  int device = 0;
};

struct gvox_map {
  std::shared_ptr<DevBuf> arena;       // descriptors, hash tables, voxel records, keys
  std::shared_ptr<GridArena> grid_arena;  // dense index grids (recycled when the last map goes)
  MapDev desc{};         // host copy
  MapDev* dev = nullptr;
  int levels = 0;
  double r0 = 0;
  // voxel counts per level: known on the host after a counted build; a
  // sync-free build leaves them on the device (counts_dev) until first asked
  mutable int64_t nvox[GVOX_MAX_LEVELS] = {};
  mutable bool counts_known = true;
  const int32_t* counts_dev = nullptr;
  const uint64_t* keys[GVOX_MAX_LEVELS] = {};
  int device = 0;
};

namespace {

gvox_status ws_reserve(gvox_ctx* ctx, int which, size_t bytes, void** out) {
  if (ctx->ws_bytes[which] < bytes) {
    size_t nb = std::max(bytes, ctx->ws_bytes[which] * 3 / 2);
    nb = align_up(nb, 1 << 20);
    if (ctx->ws[which]) {
      CK(cudaFreeAsync(ctx->ws[which], ctx->stream));
      ctx->ws[which] = nullptr;
      ctx->ws_bytes[which] = 0;
    }
    cudaError_t e = cudaMallocAsync(&ctx->ws[which], nb, ctx->stream);
    if (e != cudaSuccess) {
      char where[96];
      snprintf(where, sizeof(where), "workspace %d cudaMallocAsync(%zu bytes)", which, nb);
      return cuda_fail(e, where);
    }
    ctx->ws_bytes[which] = nb;
  }
  *out = ctx->ws[which];
  return GVOX_OK;
}

// Pinned staging for the single H2D block; waits for the previous H2D out of
// it to finish before handing it out again.
gvox_status pin_reserve(gvox_ctx* ctx, size_t bytes, void** out) {
  const int k = (ctx->pin_slot + 1) % gvox_ctx::kPinSlots;
  gvox_ctx::PinSlot& sl = ctx->pin_ring[k];
  if (!sl.done) CK(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
  if (sl.pending) {
    CK(cudaEventSynchronize(sl.done));
    sl.pending = false;
  }
  if (sl.bytes < bytes) {
    if (sl.ptr) CK(cudaFreeHost(sl.ptr));
    sl.ptr = nullptr;
    size_t nb = align_up(std::max(bytes, sl.bytes * 3 / 2), 1 << 16);
    cudaError_t e = cudaHostAlloc(&sl.ptr, nb, cudaHostAllocDefault);
    if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc");
    sl.bytes = nb;
  }
  ctx->pin_slot = k;
  *out = sl.ptr;
  return GVOX_OK;
}

// The calls' small H2D input blocks (<= 64 MiB) are read from the pinned
// staging by an SM kernel over PCIe instead of a copy-engine DMA: a bulk upload
// on another stream (the e2e pipeline's next clouds) then never delays them.
// GVOX_H2D_DMA=1 restores cudaMemcpyAsync for every block.
bool h2d_by_kernel(size_t bytes) {
  static const bool dma = std::getenv("GVOX_H2D_DMA") != nullptr;
  // blocks above GVOX_H2D_SM_MAX bytes (default 64 MiB) go by DMA: with a bulk
  // upload issued in pieces, a DMA waits for at most one piece, while SM reads
  // of a MB-sized block crawl over the busy link
  static const size_t sm_max = [] {
    const char* e = std::getenv("GVOX_H2D_SM_MAX");
    return e ? (size_t)std::max(0ll, std::atoll(e)) : (size_t)(64u << 20);
  }();
  return !dma && bytes <= sm_max;
}
gvox_status h2d_small(gvox_ctx* ctx, void* dst, const void* pinned_src, size_t bytes) {
  if (h2d_by_kernel(bytes)) {
    launch_h2d_copy(dst, pinned_src, (int64_t)bytes, ctx->stream);
    CK_LAUNCH("h2d copy");
  } else {
    CK(cudaMemcpyAsync(dst, pinned_src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  }
  return GVOX_OK;
}

// h2d_block plus a zero-fill of `zbytes` at `zdst` (a call's counters), both in
// ONE launch when the block goes by kernel
gvox_status h2d_block_zero(gvox_ctx* ctx, void* dst, const void* pinned_src, size_t bytes, void* zdst,
                           size_t zbytes) {
  gvox_ctx::PinSlot& sl = ctx->pin_ring[ctx->pin_slot];
  if (bytes && h2d_by_kernel(bytes)) {
    const H2DSeg segs[2] = {{dst, pinned_src, (int64_t)bytes}, {zdst, nullptr, (int64_t)zbytes}};
    launch_h2d_segments(segs, zbytes ? 2 : 1, ctx->stream);
    CK_LAUNCH("h2d copy");
  } else {
    if (bytes) CK(cudaMemcpyAsync(dst, pinned_src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    if (zbytes) CK(cudaMemsetAsync(zdst, 0, zbytes, ctx->stream));
  }
  // (a block that went up in the launch's parameters left the slot free)
  const bool by_param = bytes && h2d_by_kernel(bytes) && zbytes <= (size_t)(INT32_MAX / 2) &&
                        (int64_t)((bytes + 15) & ~size_t(15)) <= h2d_param_max();
  if (bytes && !by_param) {
    CK(cudaEventRecord(sl.done, ctx->stream));
    sl.pending = true;
  }
  return GVOX_OK;
}

// GVOX_LIN_EXEC_ORDER=1: linearization tiles executed grouped by target map
// (the CTAs resident together share the target's grid and records in L2); the
// results do not depend on the order.  Measured at C5: the kernel drops from
// 120.8 to 116.2 ms at full clocks (ncu launch list, r02bd), but the whole step
// then runs into the B200's power limit -- sw_power_cap, SM clocks 1886-1897
// instead of 1965 MHz -- and is no faster (r02be, 20 steps x 3 interleaved:
// 152.0 / 152.1 / 152.1 ms against 152.0 / 151.8 / 152.5), the build and the
// screening paying for the lower clock.  Same time at the cap costs more
// energy, so the batch order stays the default.
bool exec_by_target() {
  const char* e = std::getenv("GVOX_LIN_EXEC_ORDER");  // (read per call: tests switch it)
  return e != nullptr && std::atoi(e) != 0;
}

// Small batches carry their tile -> owner map in the input block (filled on the
// host; no k_tile_map launch on the critical path of an odometry-sized call).
constexpr int64_t kHostTileMapMax = 4096;
void fill_tile_map(const int32_t* tstart, int64_t n, int32_t* tm) {
  for (int64_t f = 0; f < n; ++f)
    for (int32_t t = tstart[f]; t < tstart[f + 1]; ++t) tm[t] = (int32_t)f;
}

// H2D out of the slot pin_reserve handed out last
gvox_status h2d_block(gvox_ctx* ctx, void* dst, const void* pinned_src, size_t bytes) {
  if (bytes == 0) return GVOX_OK;
  gvox_ctx::PinSlot& sl = ctx->pin_ring[ctx->pin_slot];
  gvox_status st = h2d_small(ctx, dst, pinned_src, bytes);
  if (st) return st;
  if (h2d_by_kernel(bytes) && (int64_t)bytes <= h2d_param_max()) return GVOX_OK;  // (slot free)
  CK(cudaEventRecord(sl.done, ctx->stream));
  sl.pending = true;
  return GVOX_OK;
}

// Pinned staging slot `slot` of the voxelmap build (>= bytes), once the
// previous upload out of it has completed; pin_b_upload enqueues the H2D and
// marks the slot busy until it lands.
gvox_status pin_b_reserve(gvox_ctx* ctx, int slot, size_t bytes, void** out) {
  if (!ctx->pin_b_done[slot])
    CK(cudaEventCreateWithFlags(&ctx->pin_b_done[slot], cudaEventDisableTiming));
  else
    CK(cudaEventSynchronize(ctx->pin_b_done[slot]));
  if (ctx->pin_b_bytes[slot] < bytes) {
    if (ctx->pin_b[slot]) CK(cudaFreeHost(ctx->pin_b[slot]));
    ctx->pin_b[slot] = nullptr;
    const size_t nb = align_up(std::max(bytes, ctx->pin_b_bytes[slot] * 3 / 2), 1 << 16);
    cudaError_t e = cudaHostAlloc(&ctx->pin_b[slot], nb, cudaHostAllocDefault);
    if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc");
    ctx->pin_b_bytes[slot] = nb;
  }
  *out = ctx->pin_b[slot];
  return GVOX_OK;
}
gvox_status pin_b_upload(gvox_ctx* ctx, int slot, void* dst, size_t bytes) {
  if (bytes) {
    gvox_status st = h2d_small(ctx, dst, ctx->pin_b[slot], bytes);
    if (st) return st;
  }
  CK(cudaEventRecord(ctx->pin_b_done[slot], ctx->stream));
  return GVOX_OK;
}

// two blocks out of pinned slot `slot` (at offsets 0 and off2) in one launch
gvox_status pin_b_upload2(gvox_ctx* ctx, int slot, void* dst1, size_t n1, size_t off2, void* dst2,
                          size_t n2) {
  const char* src = (const char*)ctx->pin_b[slot];
  if (h2d_by_kernel(std::max(n1, n2))) {
    const H2DSeg segs[2] = {{dst1, src, (int64_t)n1}, {dst2, src + off2, (int64_t)n2}};
    launch_h2d_segments(segs, 2, ctx->stream);
    CK_LAUNCH("h2d copy");
  } else {
    CK(cudaMemcpyAsync(dst1, src, n1, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(dst2, src + off2, n2, cudaMemcpyHostToDevice, ctx->stream));
  }
  CK(cudaEventRecord(ctx->pin_b_done[slot], ctx->stream));
  return GVOX_OK;
}

cudaEvent_t ev_get(gvox_ctx* ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Brackets the launches of one kernel group with CUDA events on the context
// stream when timing is enabled.
struct TimerScope {
  gvox_ctx* ctx;
  int which;
  cudaEvent_t a = nullptr, b = nullptr;
  TimerScope(gvox_ctx* c, int w) : ctx(c), which(w) {
    if (!ctx->timing) return;
    a = ev_get(ctx);
    b = ev_get(ctx);
    cudaEventRecord(a, ctx->stream);
  }
  ~TimerScope() {
    if (!a) return;
    cudaEventRecord(b, ctx->stream);
    ctx->ev_open[which].push_back({a, b});
  }
};

// Layout helper: a sequence of 256 B-aligned regions within one block.
struct Layout {
  size_t size = 0;
  size_t add(size_t bytes) {
    size_t off = size;
    size = align_up(size + bytes, 256);
    return off;
  }
};

}  // namespace

extern "C" {

// ------------------------------------------------------------------ context
gvox_status gvox_ctx_create(int device, void* cuda_stream, gvox_ctx** out) {
  if (!out) return fail(GVOX_ERR_INVALID, "gvox_ctx_create: out is NULL");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= ndev)
    return fail(GVOX_ERR_INVALID, "gvox_ctx_create: device %d out of range [0, %d)", device, ndev);
  DeviceGuard g(device);
  auto* c = new gvox_ctx;
  c->device = device;
  {
    size_t free_b = 0, tot_b = 0;
    if (cudaMemGetInfo(&free_b, &tot_b) == cudaSuccess) c->dense_budget = tot_b / 4;
  }
  c->stream = (cudaStream_t)cuda_stream;
  c->grid_pool->device = device;
  c->rec_pool->device = device;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;  // freed blocks stay in the pool for reuse
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  for (auto& sl : c->pin_ring) {
    e = cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      delete c;
      return cuda_fail(e, "cudaEventCreate");
    }
  }
  *out = c;
  return GVOX_OK;
}

gvox_status gvox_ctx_set_stream(gvox_ctx* ctx, void* cuda_stream) {
  if (!ctx) return fail(GVOX_ERR_INVALID, "gvox_ctx_set_stream: ctx is NULL");
  cudaStream_t next = (cudaStream_t)cuda_stream;
  if (next != ctx->stream) {
    // The grow-only workspaces (and the stream-ordered frees of the next call)
    // move to the new stream: order it after everything already queued on the
    // old one, so no kernel still reading a workspace races with its reuse.
    DeviceGuard g(ctx->device);
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev, ctx->stream) != cudaSuccess || cudaStreamWaitEvent(next, ev, 0) != cudaSuccess)
      return fail(GVOX_ERR_CUDA, "gvox_ctx_set_stream: %s", cudaGetErrorString(cudaGetLastError()));
    cudaEventDestroy(ev);  // released once the recorded work completes
    ctx->stream = next;
  }
  return GVOX_OK;
}

void gvox_ctx_destroy(gvox_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard g(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (int i = 0; i < 3; ++i)
    if (ctx->ws[i]) cudaFreeAsync(ctx->ws[i], ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  for (auto& sl : ctx->pin_ring) {
    if (sl.ptr) cudaFreeHost(sl.ptr);
    if (sl.done) cudaEventDestroy(sl.done);
  }
  for (int i = 0; i < 2; ++i) {
    if (ctx->pin_b_done[i]) cudaEventSynchronize(ctx->pin_b_done[i]);
    if (ctx->pin_b[i]) cudaFreeHost(ctx->pin_b[i]);
    if (ctx->pin_b_done[i]) cudaEventDestroy(ctx->pin_b_done[i]);
  }
  if (ctx->pin_out) cudaFreeHost(ctx->pin_out);
  if (ctx->pin_counts) cudaFreeHost(ctx->pin_counts);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (int t = 0; t < GVOX_TIMER_COUNT; ++t)
    for (auto& pr : ctx->ev_open[t]) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  delete ctx;
}

gvox_status gvox_ctx_enable_timing(gvox_ctx* ctx, int enable) {
  if (!ctx) return fail(GVOX_ERR_INVALID, "gvox_ctx_enable_timing: ctx is NULL");
  ctx->timing = enable != 0;
  return GVOX_OK;
}

gvox_status gvox_ctx_timing(gvox_ctx* ctx, double* ms, int64_t* launches, int reset) {
  if (!ctx) return fail(GVOX_ERR_INVALID, "gvox_ctx_timing: ctx is NULL");
  DeviceGuard g(ctx->device);
  for (int t = 0; t < GVOX_TIMER_COUNT; ++t) {
    for (auto& pr : ctx->ev_open[t]) {
      CK(cudaEventSynchronize(pr.second));
      float e = 0.f;
      CK(cudaEventElapsedTime(&e, pr.first, pr.second));
      ctx->timer_ms[t] += e;
      ctx->timer_launches[t] += 1;
      ctx->ev_pool.push_back(pr.first);
      ctx->ev_pool.push_back(pr.second);
    }
    ctx->ev_open[t].clear();
    if (ms) ms[t] = ctx->timer_ms[t];
    if (launches) launches[t] = ctx->timer_launches[t];
    if (reset) {
      ctx->timer_ms[t] = 0;
      ctx->timer_launches[t] = 0;
    }
  }
  return GVOX_OK;
}

// ------------------------------------------------------------------ clouds
gvox_status gvox_clouds_create(gvox_ctx* ctx, const float* mu, const float* cov,
                               const float* normals, const int64_t* offsets, int64_t count,
                               int mem, gvox_cloud** out) {
  if (!ctx || (count > 0 && (!out || !offsets)))
    return fail(GVOX_ERR_INVALID, "gvox_clouds_create: ctx/offsets/out is NULL");
  if (count < 0) return fail(GVOX_ERR_INVALID, "gvox_clouds_create: count < 0");
  if (count == 0) return GVOX_OK;
  if (offsets[0] != 0) return fail(GVOX_ERR_INVALID, "gvox_clouds_create: offsets[0] != 0");
  for (int64_t k = 0; k < count; ++k) {
    out[k] = nullptr;
    if (offsets[k + 1] < offsets[k])
      return fail(GVOX_ERR_INVALID, "gvox_cloud_create: cloud %lld has n = %lld < 0", (long long)k,
                  (long long)(offsets[k + 1] - offsets[k]));
  }
  const int64_t n = offsets[count];
  if (n > 0 && (!mu || !cov))
    return fail(GVOX_ERR_INVALID, "gvox_cloud_create: mu/cov is NULL with n = %lld", (long long)n);
  if (mem != GVOX_HOST && mem != GVOX_DEVICE)
    return fail(GVOX_ERR_INVALID, "gvox_cloud_create: mem must be GVOX_HOST or GVOX_DEVICE");
  DeviceGuard g(ctx->device);
  DebugClock dbg;
  Layout lay;
  size_t o_desc = lay.add(sizeof(CloudDev) * count);
  // chunked point records (gvox_internal.h): each cloud starts on a chunk
  std::vector<int64_t> co(count + 1, 0);
  for (int64_t k = 0; k < count; ++k) co[k + 1] = co[k] + pt_slots(offsets[k + 1] - offsets[k]);
  size_t o_pts = lay.add(16 * (size_t)co[count]);
  size_t o_flags = lay.add(32 * (size_t)count);
  // per-cloud chunk boxes (6 floats per 32 points), each cloud's run starting
  // at its own chunk 0
  std::vector<int64_t> cb_off(count + 1, 0);
  for (int64_t k = 0; k < count; ++k)
    cb_off[k + 1] = cb_off[k] + 6 * ((offsets[k + 1] - offsets[k] + kChunk - 1) / kChunk);
  size_t o_cbox = lay.add(4 * (size_t)cb_off[count]);
  size_t o_pseg = lay.add(sizeof(PackSeg) * count);
  std::shared_ptr<DevBuf> buf;
  gvox_status st = devbuf_alloc(lay.size, ctx->device, ctx->stream, &buf);
  if (st) return st;
  dbg.lap("clouds: alloc");
  char* base = (char*)buf->ptr;
  float4* P = (float4*)(base + o_pts);
  float* cbox = (float*)(base + o_cbox);
  // per-cloud statistics (see launch_cloud_pack): flag, max |C_ij|, min / max mean
  int32_t* dflags = (int32_t*)(base + o_flags);
  std::vector<int32_t> hflags(8 * (size_t)count);
  for (int64_t k = 0; k < count; ++k) {
    int32_t* st8 = hflags.data() + 8 * k;
    st8[0] = st8[1] = 0;
    st8[2] = st8[3] = st8[4] = INT32_MAX;
    st8[5] = st8[6] = st8[7] = INT32_MIN;
  }
  {
    // (small inputs through the pinned ring: no copy-engine queueing, no sync)
    void* hp = nullptr;
    st = pin_reserve(ctx, 32 * (size_t)count, &hp);
    if (st) return st;
    std::memcpy(hp, hflags.data(), 32 * (size_t)count);
    st = h2d_block(ctx, dflags, hp, 32 * (size_t)count);
    if (st) return st;
  }
  if (n > 0) {
    const float *dmu = mu, *dcov = cov, *dnrm = normals;
    if (mem == GVOX_HOST) {
      void* ws = nullptr;
      size_t bytes_in = (size_t)n * (3 + 6 + (normals ? 3 : 0)) * 4;
      st = ws_reserve(ctx, 2, bytes_in, &ws);
      if (st) return st;
      char* p = (char*)ws;
      CK(cudaMemcpyAsync(p, mu, (size_t)n * 12, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(p + n * 12, cov, (size_t)n * 24, cudaMemcpyHostToDevice, ctx->stream));
      if (normals)
        CK(cudaMemcpyAsync(p + n * 36, normals, (size_t)n * 12, cudaMemcpyHostToDevice, ctx->stream));
      dmu = (const float*)p;
      dcov = (const float*)(p + n * 12);
      dnrm = normals ? (const float*)(p + n * 36) : nullptr;
    }
    if (count <= 65535) {  // one launch for the batch (grid y = cloud)
      std::vector<PackSeg> ps(count);
      int64_t max_n = 0;
      for (int64_t k = 0; k < count; ++k) {
        const int64_t a = offsets[k], m = offsets[k + 1] - offsets[k];
        ps[k] = PackSeg{dmu + 3 * a, dcov + 6 * a, dnrm ? dnrm + 3 * a : nullptr, m, P + co[k],
                        cbox + cb_off[k], dflags + 8 * k};
        max_n = std::max(max_n, m);
      }
      {
        void* hp = nullptr;
        st = pin_reserve(ctx, sizeof(PackSeg) * count, &hp);
        if (st) return st;
        std::memcpy(hp, ps.data(), sizeof(PackSeg) * count);
        st = h2d_block(ctx, base + o_pseg, hp, sizeof(PackSeg) * count);
        if (st) return st;
      }
      launch_cloud_pack_batch((const PackSeg*)(base + o_pseg), count, max_n, ctx->stream);
    } else {
      for (int64_t k = 0; k < count; ++k) {
        int64_t a = offsets[k], m = offsets[k + 1] - offsets[k];
        if (m == 0) continue;
        launch_cloud_pack(dmu + 3 * a, dcov + 6 * a, dnrm ? dnrm + 3 * a : nullptr, m, P + co[k],
                          cbox + cb_off[k], dflags + 8 * k, ctx->stream);
      }
    }
    CK_LAUNCH("gvox_cloud_create: pack");
  }
  dbg.lap("clouds: pack enqueued");
  CK(cudaMemcpyAsync(hflags.data(), dflags, 32 * (size_t)count, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  dbg.lap("clouds: stats read back");
  for (int64_t k = 0; k < count; ++k)
    if (hflags[8 * k] & 1)
      return fail(GVOX_ERR_INVALID,
                  "gvox_cloud_create: cloud %lld has a non-finite coordinate, covariance or normal",
                  (long long)k);
  std::vector<CloudDev> descs(count);
  for (int64_t k = 0; k < count; ++k) {
    int64_t a = offsets[k], m = offsets[k + 1] - offsets[k];
    CloudDev& d = descs[k];
    d.n = m;
    d.has_normals = normals != nullptr;
    d.pad = 0;
    d.A = m ? P + co[k] : nullptr;
    d.B = m ? P + co[k] + 32 : nullptr;
    d.N = m ? P + co[k] + 64 : nullptr;
    d.chunk_box = m ? cbox + cb_off[k] : nullptr;
  }
  {
    void* hp = nullptr;
    st = pin_reserve(ctx, sizeof(CloudDev) * count, &hp);
    if (st) return st;
    std::memcpy(hp, descs.data(), sizeof(CloudDev) * count);
    st = h2d_block(ctx, base + o_desc, hp, sizeof(CloudDev) * count);
    if (st) return st;
  }
  for (int64_t k = 0; k < count; ++k) {
    auto* c = new gvox_cloud;
    c->buf = buf;
    c->desc = descs[k];
    c->dev = (CloudDev*)(base + o_desc) + k;
    c->n = descs[k].n;
    uint32_t bits = (uint32_t)hflags[8 * k + 1];
    std::memcpy(&c->cmax, &bits, 4);
    if (c->n > 0)
      for (int a = 0; a < 3; ++a) {
        c->lo[a] = ordered_to_float(hflags[8 * k + 2 + a]);
        c->hi[a] = ordered_to_float(hflags[8 * k + 5 + a]);
      }
    c->device = ctx->device;
    out[k] = c;
  }
  return GVOX_OK;
}

gvox_status gvox_cloud_create(gvox_ctx* ctx, const float* mu, const float* cov,
                              const float* normals, int64_t n, int mem, gvox_cloud** out) {
  if (!ctx || !out) return fail(GVOX_ERR_INVALID, "gvox_cloud_create: ctx/out is NULL");
  *out = nullptr;
  if (n < 0) return fail(GVOX_ERR_INVALID, "gvox_cloud_create: n = %lld < 0", (long long)n);
  const int64_t offsets[2] = {0, n};
  return gvox_clouds_create(ctx, mu, cov, normals, offsets, 1, mem, out);
}

int64_t gvox_cloud_size(const gvox_cloud* cloud) { return cloud ? cloud->n : -1; }

void gvox_cloud_destroy(gvox_cloud* cloud) { delete cloud; }

// ------------------------------------------------------------------ voxelmaps
namespace {

constexpr int64_t kBuildChunkPoints = 256 << 20;
constexpr int64_t kNoSyncBuildPoints = 4 << 20;  // chunks up to this many points build sync-free

gvox_status build_chunk(gvox_ctx* ctx, const gvox_cloud* const* clouds, int64_t count, double r0,
                        int levels, gvox_map** maps_out) {
  const int dyadic = is_dyadic(r0);
  const int L = levels;
  std::vector<int64_t> seg_start(count + 1, 0);
  for (int64_t s = 0; s < count; ++s) seg_start[s + 1] = seg_start[s] + clouds[s]->n;
  const int64_t total = seg_start[count];
  int64_t max_pts = 0;
  for (int64_t s = 0; s < count; ++s) max_pts = std::max<int64_t>(max_pts, clouds[s]->n);

  // ---- level plans from the clouds' bounding boxes (before any voxel exists).
  // Dense: an int32 grid over the level's key box when it has at most
  // kDenseBuildRatio cells per point (memory <= 4 kDenseBuildRatio B per
  // point and level), every dimension < 2^30 (the lookups rely on it) and
  // < 2^31 cells, within the chunk's dense budget (below).  Otherwise a hash
  // table sized after the voxel count is known.
  struct LevelPlan {
    bool dense = false;
    int32_t x0 = 0, y0 = 0, z0 = 0;
    uint32_t dx = 0, dy = 0, dz = 0;
    uint64_t cells = 0;
    uint64_t cap = 0;  // hash capacity
    size_t o_grid = 0, o_slots = 0, o_vox = 0, o_keys = 0;
  };
  std::vector<LevelPlan> plan((size_t)count * L);
  Layout gl;  // grid arena
  uint64_t dense_ratio = kDenseBuildRatio;  // GVOX_DENSE_RATIO env: experiments
  if (const char* e = std::getenv("GVOX_DENSE_RATIO")) dense_ratio = (uint64_t)std::max(0ll, std::atoll(e));
  for (int64_t s = 0; s < count; ++s) {
    const gvox_cloud* c = clouds[s];
    int32_t k0lo[3] = {0, 0, 0}, k0hi[3] = {0, 0, 0};
    for (int a = 0; a < 3; ++a) {
      // the device key formula (voxel_coord0), evaluated on the host; clamped
      double slo = dyadic ? (double)c->lo[a] * (1.0 / r0) : (double)c->lo[a] / r0;
      double shi = dyadic ? (double)c->hi[a] * (1.0 / r0) : (double)c->hi[a] / r0;
      double flo = std::floor(slo), fhi = std::floor(shi);
      k0lo[a] = (int32_t)std::min(std::max(flo, -1073741824.0), 1073741824.0);
      k0hi[a] = (int32_t)std::min(std::max(fhi, -1073741824.0), 1073741824.0);
    }
    for (int l = 0; l < L; ++l) {
      LevelPlan& p = plan[s * L + l];
      uint64_t cells = 1;
      int32_t lo3[3];
      int64_t n3[3];
      // NESTED boxes: every level's box is the coarsest level's key box refined
      // (x0_l = x0_c * 2^(L-1-l), d_l = d_c * 2^(L-1-l)), so a level-0 key is
      // inside the level-0 box iff its level-l key (k >> l) is inside the
      // level-l box, for every l: the linearize kernel tests the bounds once
      // per point (k_linearize.cu lookup_nested).  Costs at most 2^(L-1) - 1
      // padding cells per side of the finer grids.
      const int sc = L - 1 - l;
      for (int a = 0; a < 3; ++a) {
        const int32_t clo = k0lo[a] >> (L - 1), chi = k0hi[a] >> (L - 1);
        lo3[a] = clo * (1 << sc);  // |clo| <= 2^30 >> (L - 1): no overflow
        n3[a] = ((int64_t)chi - clo + 1) << sc;
      }
      const bool dims_ok = n3[0] < (1 << 30) && n3[1] < (1 << 30) && n3[2] < (1 << 30);
      // (saturating: a product above 2^62 is far beyond any dense grid)
      for (int a = 0; a < 3; ++a)
        cells = (dims_ok && cells <= (1ull << 32)) ? cells * (uint64_t)n3[a] : (1ull << 62);
      if (c->n > 0 && dims_ok && cells <= dense_ratio * (uint64_t)c->n &&
          cells < (1ull << 31)) {
        p.dense = true;
        p.x0 = lo3[0]; p.y0 = lo3[1]; p.z0 = lo3[2];
        p.dx = n3[0]; p.dy = n3[1]; p.dz = n3[2];
        p.cells = cells;
      }
    }
  }
  // Dense grids trade HBM for one-load lookups; keep the chunk's grids within
  // a budget (a quarter of the device memory, GVOX_DENSE_BUDGET_MB overrides)
  // by demoting the largest grids to hash levels.
  {
    uint64_t total_cells = 0;
    for (const LevelPlan& p : plan)
      if (p.dense) total_cells += p.cells;
    uint64_t budget = ctx->dense_budget;
    if (const char* e = std::getenv("GVOX_DENSE_BUDGET_MB")) budget = (uint64_t)std::atoll(e) << 20;
    if (4 * total_cells > budget) {
      std::vector<size_t> idx;
      for (size_t i = 0; i < plan.size(); ++i)
        if (plan[i].dense) idx.push_back(i);
      std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return plan[a].cells > plan[b].cells; });
      for (size_t i : idx) {
        if (4 * total_cells <= budget) break;
        total_cells -= plan[i].cells;
        plan[i] = LevelPlan{};
      }
    }
    for (LevelPlan& p : plan)
      if (p.dense) p.o_grid = gl.add(p.cells * 4);
  }
  DebugClock dbg;
  dbg.lap("plan");
  std::shared_ptr<GridArena> grid_arena;
  bool grid_fresh = true;
  gvox_status st = grid_arena_take(ctx->grid_pool, gl.size, ctx->device, ctx->stream, &grid_arena,
                                   &grid_fresh);
  dbg.lap("grid alloc");
  if (st) return st;
  char* gb = (char*)grid_arena->ptr;
  // every cell -1 (empty); a recycled arena already is
  if (gl.size && grid_fresh) CK(cudaMemsetAsync(gb, 0xFF, gl.size, ctx->stream));

  // ---- sync-free or counted.  A small chunk (odometry frames, keyframe maps:
  // <= kNoSyncBuildPoints points) sizes every buffer by the bound "at most one
  // voxel per point and level" before the insert, so the host never waits for
  // the GPU: the accumulators are zeroed by the insert as voxels are created,
  // finalize and the grid reset read the counts on the device, and the range
  // error is decided from the clouds' bounding boxes on the host (the level-0
  // keys are the widest; floor is monotone, so the box corners decide it
  // exactly).  A large chunk reads the counts back once and sizes exactly.
  bool nosync = total <= kNoSyncBuildPoints;
  if (const char* e = std::getenv("GVOX_BUILD_NOSYNC")) nosync = std::atoi(e) != 0;
  // Lifted accumulation (level 0 from the points, every coarser level from the
  // voxels below it, k_build_lift) pays on large chunks (C5: 17.96 -> 14.95 ms);
  // small ones (odometry frames) are launch-bound and accumulate every level
  // from the points in one kernel.  GVOX_BUILD_LIFT=0/1 overrides.
  bool lift = L > 1 && total > kNoSyncBuildPoints;
  if (const char* e = std::getenv("GVOX_BUILD_LIFT")) lift = L > 1 && std::atoi(e) != 0;
  for (int64_t s = 0; s < count; ++s) {
    const gvox_cloud* c = clouds[s];
    if (c->n <= 0) continue;
    for (int a = 0; a < 3; ++a) {
      const double slo = dyadic ? (double)c->lo[a] * (1.0 / r0) : (double)c->lo[a] / r0;
      const double shi = dyadic ? (double)c->hi[a] * (1.0 / r0) : (double)c->hi[a] / r0;
      if (std::floor(slo) < -1048576.0 || std::floor(shi) >= 1048576.0)
        return fail(GVOX_ERR_RANGE,
                    "gvox_create_voxelmap: a voxel key is outside [-2^20, 2^20) (r0 = %g)", r0);
    }
  }

  // ---- phase 1 workspace (workspace 0): hash-level temp tables, keys, slots
  std::vector<uint64_t> tcap(count);
  Layout lay;
  std::vector<size_t> o_tmp(count), o_keys(count);
  std::vector<int> nhash(count, 0);
  for (int64_t s = 0; s < count; ++s) {
    tcap[s] = pow2_at_least(std::max<uint64_t>(16, 2 * (uint64_t)clouds[s]->n));
    for (int l = 0; l < L; ++l) nhash[s] += !plan[s * L + l].dense;
    o_tmp[s] = lay.add(tcap[s] * 16 * nhash[s]);
  }
  const size_t tmp_bytes = lay.size;  // temp tables first: one 0xFF memset
  for (int64_t s = 0; s < count; ++s) o_keys[s] = lay.add((size_t)clouds[s]->n * 8 * L);
  size_t o_pslot = lay.add((size_t)total * L * 4);
  // the counters and the insert descriptors: ONE upload (zeros, then BuildSeg[])
  size_t o_cnt = lay.add((size_t)count * L * 4 + 4);
  size_t o_bseg = lay.add(sizeof(BuildSeg) * count);
  const size_t ins_bytes = o_bseg + sizeof(BuildSeg) * count - o_cnt;
  void* ws0 = nullptr;
  st = ws_reserve(ctx, 0, lay.size, &ws0);
  if (st) return st;
  dbg.lap("ws0");
  char* b0 = (char*)ws0;
  int32_t* d_cnt = (int32_t*)(b0 + o_cnt);
  int32_t* d_err = d_cnt + count * L;

  std::vector<BuildSeg> bseg(count);
  for (int64_t s = 0; s < count; ++s) {
    BuildSeg& g = bseg[s];
    std::memset(&g, 0, sizeof(g));
    g.A = clouds[s]->desc.A;
    g.n = clouds[s]->n;
    g.pl_offset = seg_start[s];
    g.pl_stride = total;
    g.tmp_mask = tcap[s] - 1;
    g.tmp_shift = shift_for_capacity(tcap[s]);
    g.lift = lift ? 1 : 0;
    int hslot = 0;
    for (int l = 0; l < L; ++l) {
      const LevelPlan& p = plan[s * L + l];
      LevelBox& bx = g.box[l];
      bx.dense = p.dense;
      if (p.dense) {
        bx.x0 = p.x0; bx.y0 = p.y0; bx.z0 = p.z0;
        bx.dx = p.dx; bx.dy = p.dy; bx.dz = p.dz;
        bx.syz = p.dy * p.dz;
        bx.grid = (int32_t*)(gb + p.o_grid);
      } else {
        g.tmp_slots[l] = (ulonglong2*)(b0 + o_tmp[s]) + tcap[s] * hslot++;
      }
      g.keys_by_idx[l] = (uint64_t*)(b0 + o_keys[s]) + (size_t)clouds[s]->n * l;
    }
    g.counter = d_cnt + s * L;
  }
  if (tmp_bytes) CK(cudaMemsetAsync(b0, 0xFF, tmp_bytes, ctx->stream));

  // voxel capacity of every (map, level): the point count (sync-free) or the
  // exact count (counted, after the readback)
  std::vector<int64_t> vcap((size_t)count * L);
  std::vector<int32_t> hcnt((size_t)count * L + 1, 0);
  auto launch_insert = [&](bool upload) -> gvox_status {
    if (upload) {
      void* hp = nullptr;
      gvox_status st2 = pin_b_reserve(ctx, 0, ins_bytes, &hp);
      if (st2) return st2;
      std::memset(hp, 0, o_bseg - o_cnt);  // the voxel counters and the range flag start at 0
      std::memcpy((char*)hp + (o_bseg - o_cnt), bseg.data(), sizeof(BuildSeg) * count);
      st2 = pin_b_upload(ctx, 0, b0 + o_cnt, ins_bytes);
      if (st2) return st2;
    }
    TimerScope ts(ctx, GVOX_TIMER_BUILD);
    launch_build_insert((const BuildSeg*)(b0 + o_bseg), count, max_pts, L, r0, dyadic,
                        (int32_t*)(b0 + o_pslot), d_err, ctx->stream);
    CK_LAUNCH("voxelmap insert");
    return GVOX_OK;
  };
  if (nosync) {
    for (int64_t s = 0; s < count; ++s)
      for (int l = 0; l < L; ++l) vcap[s * L + l] = clouds[s]->n;
  } else {
    st = launch_insert(true);
    if (st) return st;
    CK(cudaMemcpyAsync(hcnt.data(), d_cnt, ((size_t)count * L + 1) * 4, cudaMemcpyDeviceToHost,
                       ctx->stream));
    dbg.lap("insert enqueued");
    CK(cudaStreamSynchronize(ctx->stream));
    dbg.lap("insert sync");
    if (hcnt[(size_t)count * L])
      return fail(GVOX_ERR_RANGE,
                  "gvox_create_voxelmap: a voxel key is outside [-2^20, 2^20) (r0 = %g)", r0);
    for (int64_t q = 0; q < count * L; ++q) vcap[q] = hcnt[q];
  }

  // ---- record arena: build metadata (uploaded as ONE pinned H2D: map
  // descriptors, grid-reset table, accumulate / finalize segments, voxel
  // counts), hash tables, voxel records, keys
  Layout al;
  int64_t total_vox = 0;
  const size_t o_descs = al.add(sizeof(MapDev) * count);
  const size_t o_reset = al.add(sizeof(ResetSeg) * count * L);
  const size_t o_aseg = al.add(sizeof(AccumSeg) * count);
  const size_t o_fseg = al.add(sizeof(FinalSeg) * count * L);
  const size_t o_counts = al.add((size_t)count * L * 4);  // the maps' voxel counts
  const size_t meta_end = al.size;
  const size_t idx_begin = al.size;  // final hash tables: one 0xFF memset
  for (int64_t s = 0; s < count; ++s)
    for (int l = 0; l < L; ++l) {
      LevelPlan& p = plan[s * L + l];
      if (!p.dense) {
        p.cap = pow2_at_least(std::max<uint64_t>(2, 2 * (uint64_t)vcap[s * L + l]));
        p.o_slots = al.add(p.cap * 16);
      }
    }
  const size_t idx_end = al.size;
  for (int64_t s = 0; s < count; ++s)
    for (int l = 0; l < L; ++l) {
      const int64_t V = vcap[s * L + l];
      LevelPlan& p = plan[s * L + l];
      p.o_vox = al.add((size_t)(V + 1) * 48);  // + the all-zero sentinel record at index -1
      p.o_keys = al.add((size_t)V * 8);
      total_vox += V;
    }
  std::shared_ptr<DevBuf> arena;
  // (small, sync-free builds recycle their record arenas; large ones free them)
  st = devbuf_alloc(al.size, ctx->device, ctx->stream, &arena, nosync ? ctx->rec_pool : nullptr);
  if (st) return st;
  dbg.lap("record alloc");
  char* ab = (char*)arena->ptr;
  const int32_t* d_counts = (const int32_t*)(ab + o_counts);
  // ---- phase 2/3 workspace (workspace 1): acc [total_vox][10]
  Layout l1;
  size_t o_acc = l1.add((size_t)total_vox * 80);
  void* ws1 = nullptr;
  st = ws_reserve(ctx, 1, l1.size, &ws1);
  if (st) return st;
  dbg.lap("ws1");
  char* b1 = (char*)ws1;
  if (!nosync) CK(cudaMemsetAsync(b1 + o_acc, 0, (size_t)total_vox * 80, ctx->stream));
  if (idx_end > idx_begin) CK(cudaMemsetAsync(ab + idx_begin, 0xFF, idx_end - idx_begin, ctx->stream));

  // the metadata is written straight into the pinned block that uploads it
  // (no staging vectors and copies: this host work sits between the count
  // readback and the accumulation, with the GPU idle, in counted builds)
  const size_t meta_bytes = meta_end - o_descs;
  const size_t ins_off = align_up(meta_bytes, 256);
  void* hp = nullptr;
  st = pin_b_reserve(ctx, 1, nosync ? ins_off + ins_bytes : meta_bytes, &hp);
  if (st) return st;
  char* const h = (char*)hp - o_descs;  // the pinned block mirrors [o_descs, meta_end)
  AccumSeg* const aseg = (AccumSeg*)(h + o_aseg);
  FinalSeg* const fseg = (FinalSeg*)(h + o_fseg);
  MapDev* const mdesc = (MapDev*)(h + o_descs);
  int64_t vacc = 0;
  for (int64_t s = 0; s < count; ++s) {
    const gvox_cloud* c = clouds[s];
    // fixed-point: F fraction bits so that n * 2^F <= 2^61 (voxel sums fit in
    // int64) and F <= 46 (one value fits the kernel's two 32-bit REDUX chunks)
    int nb = 0;
    while ((1ll << nb) <= c->n) ++nb;  // 2^nb > n
    const int F = std::min(61 - nb, 46);
    int ec = 0;
    if (c->cmax > 0.f) {
      std::frexp((double)c->cmax, &ec);  // cmax < 2^ec
    }
    AccumSeg& a = aseg[s];
    std::memset(&a, 0, sizeof(a));
    a.A = c->desc.A;
    a.B = c->desc.B;
    a.N = c->desc.N;
    a.n = c->n;
    a.pl_offset = seg_start[s];
    a.pl_stride = total;
    a.cov_scale = std::ldexp(1.0, F - ec);
    MapDev& md = mdesc[s];
    std::memset(&md, 0, sizeof(md));
    md.levels = L;
    md.dyadic = dyadic;
    md.r0 = r0;
    md.inv_r0 = 1.0 / r0;
    {
      const float rmax = (float)std::ldexp(r0, L - 1);
      for (int a3 = 0; a3 < 3; ++a3) {
        md.box_lo[a3] = c->n > 0 ? c->lo[a3] - rmax : INFINITY;
        md.box_hi[a3] = c->n > 0 ? c->hi[a3] + rmax : -INFINITY;
      }
      md.box_lo[3] = md.box_hi[3] = 0.f;
    }
    for (int l = 0; l < L; ++l) {
      const int64_t V = vcap[s * L + l];
      const double r = std::ldexp(r0, l);
      const LevelPlan& p = plan[s * L + l];
      a.acc_offset[l] = vacc;
      // lifted builds: one offset scale for every level (the coarsest level's),
      // so k_build_lift moves a voxel's sums into its parent exactly
      a.mu_scale[l] = std::ldexp(1.0, F) / (lift ? std::ldexp(r0, L - 1) : r);
      if (nosync) {
        bseg[s].acc = (unsigned long long*)(b1 + o_acc);
        bseg[s].acc_offset[l] = vacc;
      }
      FinalSeg& f = fseg[s * L + l];
      std::memset(&f, 0, sizeof(f));
      f.acc_offset = vacc;
      f.nvox = d_cnt + s * L + l;  // the insert's counter (this build's workspace)
      f.nvox_out = const_cast<int32_t*>(d_counts) + s * L + l;  // the map's copy
      f.keys_by_idx = bseg[s].keys_by_idx[l];
      f.r = r;
      f.mu_scale = a.mu_scale[l];
      f.cov_scale = a.cov_scale;
      f.slots = p.dense ? nullptr : (ulonglong2*)(ab + p.o_slots);  // dense: grid built in phase 1
      f.mask = p.dense ? 0 : p.cap - 1;
      f.shift = p.dense ? 64 : shift_for_capacity(p.cap);
      f.dense = p.dense;
      f.grid = nullptr;
      f.vox = (float4*)(ab + p.o_vox) + 3;  // record -1: the zero sentinel (written by finalize)
      f.keys_out = (uint64_t*)(ab + p.o_keys);
      MapLevelDev& lv = md.lv[l];
      lv.slots = f.slots;
      lv.vox = f.vox;
      lv.mask = f.mask;
      lv.shift = f.shift;
      lv.grid = p.dense ? (const int32_t*)(gb + p.o_grid) : nullptr;
      lv.dense = p.dense;
      lv.x0 = p.x0; lv.y0 = p.y0; lv.z0 = p.z0;
      lv.dx = p.dx; lv.dy = p.dy; lv.dz = p.dz;
      lv.syz = p.dy * p.dz;
      lv.r = r;
      lv.inv_r = 1.0 / r;
      lv.nvox = nosync ? -1 : V;  // (host-side information only; -1: on the device)
      vacc += V;
    }
  }
  int64_t max_vox = 0;
  for (int64_t q = 0; q < count * L; ++q) max_vox = std::max<int64_t>(max_vox, vcap[q]);
  {
    // reset table of the dense levels (GridArena: recycling the grids)
    ResetSeg* const rseg = (ResetSeg*)(h + o_reset);
    for (int64_t q = 0; q < count * L; ++q) {
      const LevelPlan& p = plan[q];
      ResetSeg& r = rseg[q];
      std::memset(&r, 0, sizeof(r));
      if (!p.dense) continue;
      r.keys = fseg[q].keys_out;
      r.grid = (int32_t*)(gb + p.o_grid);
      r.nvox = d_counts + q;
      r.x0 = p.x0; r.y0 = p.y0; r.z0 = p.z0;
      r.dy = p.dy; r.dz = p.dz;
    }
    // sync-free builds: the metadata and the insert descriptors (+ zeroed
    // counters) go up in ONE launch out of one pinned slot
    std::memcpy(h + o_counts, hcnt.data(), (size_t)count * L * 4);  // counted: the exact counts
    if (nosync) {
      char* hi = (char*)hp + ins_off;
      std::memset(hi, 0, o_bseg - o_cnt);  // the voxel counters and the range flag start at 0
      std::memcpy(hi + (o_bseg - o_cnt), bseg.data(), sizeof(BuildSeg) * count);
      st = pin_b_upload2(ctx, 1, ab + o_descs, meta_bytes, ins_off, b0 + o_cnt, ins_bytes);
    } else {
      st = pin_b_upload(ctx, 1, ab + o_descs, meta_bytes);
    }
    if (st) return st;
    grid_arena->rec = arena;
    grid_arena->reset = (const ResetSeg*)(ab + o_reset);
    grid_arena->nreset = count * L;
    grid_arena->max_vox = max_vox;
  }
  if (nosync) {
    st = launch_insert(false);  // (uploaded above; its accumulator zeroing needs bseg's acc fields)
    if (st) return st;
    // (the maps' counts: copied from the insert's counters by the finalize)
    dbg.lap("insert enqueued (sync-free)");
  }
  {
    TimerScope ts(ctx, GVOX_TIMER_BUILD);
    launch_build_accum((const BuildSeg*)(b0 + o_bseg), (const AccumSeg*)(ab + o_aseg), count,
                       max_pts, L, r0, dyadic, (const int32_t*)(b0 + o_pslot),
                       (unsigned long long*)(b1 + o_acc), ctx->stream);
  }
  CK_LAUNCH("voxelmap accumulate");
  {
    std::vector<int64_t> maxv(L, 0);
    for (int64_t s2 = 0; s2 < count; ++s2)
      for (int l = 0; l < L; ++l) maxv[l] = std::max<int64_t>(maxv[l], vcap[s2 * L + l]);
    TimerScope ts(ctx, GVOX_TIMER_BUILD);
    if (lift)
      launch_build_lift((const BuildSeg*)(b0 + o_bseg), (const AccumSeg*)(ab + o_aseg), count, L,
                        maxv.data(), r0, (unsigned long long*)(b1 + o_acc), ctx->stream);
  }
  CK_LAUNCH("voxelmap lift");
  {
    TimerScope ts(ctx, GVOX_TIMER_BUILD);
    launch_build_finalize((const FinalSeg*)(ab + o_fseg), count * L, max_vox,
                          (const unsigned long long*)(b1 + o_acc), ctx->stream);
  }
  CK_LAUNCH("voxelmap finalize");
  // (the stream orders the next chunk's reuse of the workspaces after this one)
  dbg.lap("accum/finalize enqueued");
  for (int64_t s = 0; s < count; ++s) {
    auto* m = new gvox_map;
    m->arena = arena;
    m->grid_arena = grid_arena;
    m->desc = mdesc[s];
    m->dev = (MapDev*)(ab + o_descs) + s;
    m->levels = L;
    m->r0 = r0;
    m->device = ctx->device;
    m->counts_dev = d_counts + s * L;
    m->counts_known = !nosync;
    for (int l = 0; l < L; ++l) {
      m->nvox[l] = nosync ? -1 : hcnt[s * L + l];
      m->keys[l] = fseg[s * L + l].keys_out;
    }
    maps_out[s] = m;
  }
  return GVOX_OK;
}

}  // namespace

gvox_status gvox_create_voxelmaps(gvox_ctx* ctx, const gvox_cloud* const* clouds, int64_t count,
                                  double r0, int levels, gvox_map** maps_out) {
  if (!ctx || (!clouds && count > 0) || (!maps_out && count > 0))
    return fail(GVOX_ERR_INVALID, "gvox_create_voxelmaps: NULL argument");
  if (count < 0) return fail(GVOX_ERR_INVALID, "gvox_create_voxelmaps: count < 0");
  if (!(r0 > 0.0) || !std::isfinite(r0))
    return fail(GVOX_ERR_INVALID, "gvox_create_voxelmap: r0 = %g must be finite and > 0", r0);
  if (levels < 1 || levels > GVOX_MAX_LEVELS)
    return fail(GVOX_ERR_INVALID, "gvox_create_voxelmap: levels = %d outside [1, %d]", levels,
                GVOX_MAX_LEVELS);
  for (int64_t s = 0; s < count; ++s) {
    if (!clouds[s]) return fail(GVOX_ERR_INVALID, "gvox_create_voxelmaps: clouds[%lld] is NULL", (long long)s);
    maps_out[s] = nullptr;
  }
  DeviceGuard g(ctx->device);
  int64_t s0 = 0;
  while (s0 < count) {
    int64_t s1 = s0, pts = 0;
    // a chunk: <= kBuildChunkPoints points and <= 65535 / levels maps (grid rows)
    while (s1 < count && (s1 == s0 || (pts + clouds[s1]->n <= kBuildChunkPoints &&
                                       (s1 - s0 + 1) * levels <= 65535)))
      pts += clouds[s1++]->n;
    gvox_status st = build_chunk(ctx, clouds + s0, s1 - s0, r0, levels, maps_out + s0);
    if (st) {
      for (int64_t s = 0; s < s0; ++s) {
        delete maps_out[s];
        maps_out[s] = nullptr;
      }
      return st;
    }
    s0 = s1;
  }
  return GVOX_OK;
}

gvox_status gvox_create_voxelmap(gvox_ctx* ctx, const gvox_cloud* cloud, double r0, int levels,
                                 gvox_map** out) {
  if (!cloud || !out) return fail(GVOX_ERR_INVALID, "gvox_create_voxelmap: NULL argument");
  return gvox_create_voxelmaps(ctx, &cloud, 1, r0, levels, out);
}

// The voxel counts of a sync-free build live on the device until first asked.
gvox_status resolve_counts(const gvox_map* map) {
  if (map->counts_known) return GVOX_OK;
  DeviceGuard g(map->device);
  int32_t c[GVOX_MAX_LEVELS] = {};
  const cudaStream_t st = map->arena->stream;  // the building stream: after the build
  CK(cudaMemcpyAsync(c, map->counts_dev, 4 * map->levels, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int l = 0; l < map->levels; ++l) map->nvox[l] = c[l];
  map->counts_known = true;
  return GVOX_OK;
}

gvox_status gvox_voxelmap_info(const gvox_map* map, int level, int64_t* num_voxels,
                               double* resolution) {
  if (!map) return fail(GVOX_ERR_INVALID, "gvox_voxelmap_info: map is NULL");
  if (level < 0 || level >= map->levels)
    return fail(GVOX_ERR_INVALID, "gvox_voxelmap_info: level %d outside [0, %d)", level, map->levels);
  if (num_voxels) {
    gvox_status st = resolve_counts(map);
    if (st) return st;
    *num_voxels = map->nvox[level];
  }
  if (resolution) *resolution = std::ldexp(map->r0, level);
  return GVOX_OK;
}

int gvox_voxelmap_levels(const gvox_map* map) { return map ? map->levels : -1; }

gvox_status gvox_voxelmap_export(gvox_ctx* ctx, const gvox_map* map, int level, int64_t* keys,
                                 double* means, double* covs, int32_t* counts) {
  if (!ctx || !map) return fail(GVOX_ERR_INVALID, "gvox_voxelmap_export: NULL argument");
  if (level < 0 || level >= map->levels)
    return fail(GVOX_ERR_INVALID, "gvox_voxelmap_export: level %d outside [0, %d)", level, map->levels);
  DeviceGuard g(ctx->device);
  gvox_status st0 = resolve_counts(map);
  if (st0) return st0;
  const int64_t V = map->nvox[level];
  std::vector<uint64_t> k(V);
  std::vector<float4> v(3 * V);
  if (V) {
    CK(cudaMemcpyAsync(k.data(), map->keys[level], 8 * V, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(v.data(), map->desc.lv[level].vox, 48 * V, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  std::vector<int64_t> ord(V);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return k[a] < k[b]; });
  const double r = std::ldexp(map->r0, level);
  for (int64_t i = 0; i < V; ++i) {
    int64_t j = ord[i];
    uint64_t key = k[j];
    int64_t kk[3] = {(int64_t)((key >> 42) & 0x1FFFFF) - kKeyHalf,
                     (int64_t)((key >> 21) & 0x1FFFFF) - kKeyHalf, (int64_t)(key & 0x1FFFFF) - kKeyHalf};
    const float4 a = v[3 * j], b = v[3 * j + 1], c = v[3 * j + 2];
    if (keys) keys[i] = (int64_t)key;
    if (means) {
      const float off[3] = {a.x, a.y, a.z};
      for (int d = 0; d < 3; ++d) means[3 * i + d] = ((double)kk[d] + 0.5) * r + (double)off[d];
    }
    if (covs) {
      const float cv[6] = {a.w, b.x, b.z, b.y, b.w, c.x};  // record: {xy, yy, xz, yz}
      for (int d = 0; d < 6; ++d) covs[6 * i + d] = cv[d];
    }
    if (counts) {
      int32_t cnt;
      std::memcpy(&cnt, &c.y, 4);
      counts[i] = cnt;
    }
  }
  return GVOX_OK;
}

gvox_status gvox_voxelmap_lookup(gvox_ctx* ctx, const gvox_map* map, int level, const double* q,
                                 int64_t n, int64_t* keys_out, int mem) {
  if (!ctx || !map || (n > 0 && (!q || !keys_out)))
    return fail(GVOX_ERR_INVALID, "gvox_voxelmap_lookup: NULL argument");
  if (n < 0) return fail(GVOX_ERR_INVALID, "gvox_voxelmap_lookup: n < 0");
  if (level < 0 || level >= map->levels)
    return fail(GVOX_ERR_INVALID, "gvox_voxelmap_lookup: level %d outside [0, %d)", level, map->levels);
  if (n == 0) return GVOX_OK;
  DeviceGuard g(ctx->device);
  const double* dq = q;
  int64_t* dout = keys_out;
  if (mem == GVOX_HOST) {
    void* ws = nullptr;
    gvox_status st = ws_reserve(ctx, 2, (size_t)n * 32 + 256, &ws);
    if (st) return st;
    dq = (const double*)ws;
    dout = (int64_t*)((char*)ws + align_up((size_t)n * 24, 256));
    CK(cudaMemcpyAsync((void*)dq, q, (size_t)n * 24, cudaMemcpyHostToDevice, ctx->stream));
  }
  launch_lookup(map->dev, level, dq, n, dout, ctx->stream);
  CK_LAUNCH("gvox_voxelmap_lookup");
  if (mem == GVOX_HOST) {
    CK(cudaMemcpyAsync(keys_out, dout, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return GVOX_OK;
}

void gvox_map_destroy(gvox_map* map) { delete map; }

void gvox_maps_destroy(gvox_map* const* maps, int64_t count) {
  if (!maps) return;
  for (int64_t i = 0; i < count; ++i) delete maps[i];
}

// ------------------------------------------------------------------ overlap
namespace {

// Shared by gvox_overlap (counts) and gvox_overlap_select (decisions).
gvox_status overlap_impl(const char* fn, gvox_ctx* ctx, const gvox_cloud* const* clouds,
                         int64_t num_clouds, const gvox_map* const* maps, int64_t num_maps,
                         const gvox_pair* pairs, int64_t num_pairs, const double* poses,
                         int64_t num_poses, int level, int32_t* counts, uint8_t* selected,
                         int32_t num, int32_t den, int mem) {
  if (!ctx) return fail(GVOX_ERR_INVALID, "%s: ctx is NULL", fn);
  if (num_pairs < 0) return fail(GVOX_ERR_INVALID, "%s: num_pairs < 0", fn);
  if (num_pairs == 0) return GVOX_OK;
  if (!clouds || !maps || !pairs || !poses || !(counts || selected))
    return fail(GVOX_ERR_INVALID, "%s: NULL argument", fn);
  if (mem != GVOX_HOST && mem != GVOX_DEVICE)
    return fail(GVOX_ERR_INVALID, "%s: mem must be GVOX_HOST or GVOX_DEVICE", fn);
  if (selected && (num < 0 || den <= 0))
    return fail(GVOX_ERR_INVALID, "%s: threshold num = %d, den = %d (need num >= 0, den > 0)", fn,
                num, den);
  if (num_pairs > INT32_MAX) return fail(GVOX_ERR_INVALID, "%s: more than 2^31 pairs", fn);
  for (int64_t p = 0; p < num_pairs; ++p) {
    const gvox_pair& q = pairs[p];
    if (q.source_cloud < 0 || q.source_cloud >= num_clouds || !clouds[q.source_cloud])
      return fail(GVOX_ERR_INVALID, "%s: pair %lld: source_cloud %d out of range [0, %lld)", fn,
                  (long long)p, q.source_cloud, (long long)num_clouds);
    if (q.target_map < 0 || q.target_map >= num_maps || !maps[q.target_map])
      return fail(GVOX_ERR_INVALID, "%s: pair %lld: target_map %d out of range [0, %lld)", fn,
                  (long long)p, q.target_map, (long long)num_maps);
    if (q.pose_i < 0 || q.pose_i >= num_poses || q.pose_j < 0 || q.pose_j >= num_poses)
      return fail(GVOX_ERR_INVALID, "%s: pair %lld: pose index out of range [0, %lld)", fn,
                  (long long)p, (long long)num_poses);
    if (level < 0 || level >= maps[q.target_map]->levels)
      return fail(GVOX_ERR_INVALID, "%s: pair %lld: level %d outside the target map's [0, %d)", fn,
                  (long long)p, level, maps[q.target_map]->levels);
  }
  for (int64_t i = 0; i < num_poses; ++i)
    if (!finite_pose(poses + 12 * i))
      return fail(GVOX_ERR_INVALID, "%s: pose %lld is not finite", fn, (long long)i);
  DeviceGuard g(ctx->device);
  int64_t total_pts = 0;
  bool all_dense = true, all_dyadic = true;
  for (int64_t p = 0; p < num_pairs; ++p) {
    total_pts += clouds[pairs[p].source_cloud]->n;
    all_dyadic = all_dyadic && maps[pairs[p].target_map]->desc.dyadic;
    all_dense = all_dense && maps[pairs[p].target_map]->desc.lv[level].dense;
  }
  // counts: tiles of 256 * ppt source points, >= ~8 waves of 8 CTAs per SM
  // (selection: one CTA per pair, no tiles)
  int ppt = 4;  // the kernel handles U points per thread per iteration
  while (ppt < 32 && total_pts / ((int64_t)256 * ppt * 2) >= 148 * 8 * 8) ppt *= 2;
  const int tile_pts = 256 * ppt;
  std::vector<int32_t> tstart(counts ? num_pairs + 1 : 1, 0);
  if (counts)
    for (int64_t p = 0; p < num_pairs; ++p) {
      int64_t n = clouds[pairs[p].source_cloud]->n;
      int64_t nt = tstart[p] + (n + tile_pts - 1) / tile_pts;
      if (nt > INT32_MAX) return fail(GVOX_ERR_INVALID, "%s: more than 2^31 tiles", fn);
      tstart[p + 1] = (int32_t)nt;
    }
  const int64_t T = tstart.back();
  // ---- one serialized input block
  Layout lay;
  size_t o_pose = lay.add(96 * num_poses);
  size_t o_pair = lay.add(sizeof(PairDev) * num_pairs);
  size_t o_ts = lay.add(4 * tstart.size());
  const bool host_tm = counts && T <= kHostTileMapMax;  // (selection: no tiles)
  size_t o_tm = lay.add(host_tm ? 4 * (size_t)T : 0);
  size_t o_cl = lay.add(8 * num_clouds);
  size_t o_mp = lay.add(8 * num_maps);
  size_t in_bytes = lay.size;
  void* pin = nullptr;
  gvox_status st = pin_reserve(ctx, in_bytes, &pin);
  if (st) return st;
  char* hp = (char*)pin;
  std::memcpy(hp + o_pose, poses, 96 * num_poses);
  std::memcpy(hp + o_pair, pairs, sizeof(PairDev) * num_pairs);
  std::memcpy(hp + o_ts, tstart.data(), 4 * tstart.size());
  if (host_tm) fill_tile_map(tstart.data(), num_pairs, (int32_t*)(hp + o_tm));
  for (int64_t i = 0; i < num_clouds; ++i) ((const CloudDev**)(hp + o_cl))[i] = clouds[i] ? clouds[i]->dev : nullptr;
  for (int64_t i = 0; i < num_maps; ++i) ((const MapDev**)(hp + o_mp))[i] = maps[i] ? maps[i]->dev : nullptr;
  Layout wl;
  size_t o_in = wl.add(in_bytes);
  size_t o_tp = wl.add(host_tm ? 0 : 4 * (size_t)std::max<int64_t>(T, 1));
  size_t o_out = wl.add(4 * num_pairs);
  void* ws = nullptr;
  st = ws_reserve(ctx, 0, wl.size, &ws);
  if (st) return st;
  char* wb = (char*)ws;
  // the counts start at zero: zeroed by the same launch that uploads the block
  int32_t* const dcounts0 = counts ? (mem == GVOX_DEVICE ? counts : (int32_t*)(wb + o_out)) : nullptr;
  st = h2d_block_zero(ctx, wb + o_in, hp, in_bytes, dcounts0, counts ? 4 * (size_t)num_pairs : 0);
  if (st) return st;
  char* din = wb + o_in;
  const CloudDev* const* dcl = (const CloudDev* const*)(din + o_cl);
  const MapDev* const* dmp = (const MapDev* const*)(din + o_mp);
  const PairDev* dpairs = (const PairDev*)(din + o_pair);
  const double* dposes = (const double*)(din + o_pose);
  size_t out_bytes;
  void* dout;
  if (counts) {
    int32_t* dcounts = dcounts0;
    int32_t* dtm = host_tm ? (int32_t*)(din + o_tm) : (int32_t*)(wb + o_tp);
    if (!host_tm) launch_tile_map((const int32_t*)(din + o_ts), num_pairs, dtm, ctx->stream);
    TimerScope ts(ctx, GVOX_TIMER_OVERLAP);
    launch_overlap(dcl, dmp, dpairs, (const int32_t*)(din + o_ts), num_pairs, T, tile_pts, dposes,
                   level, dtm, dcounts, all_dense, ctx->stream);
    dout = dcounts;
    out_bytes = 4 * num_pairs;
  } else {
    uint8_t* dsel = mem == GVOX_DEVICE ? selected : (uint8_t*)(wb + o_out);
    TimerScope ts(ctx, GVOX_TIMER_OVERLAP);
    launch_overlap_select(dcl, dmp, dpairs, num_pairs, dposes, level, num, den, dsel, all_dense,
                          all_dyadic, ctx->stream);
    dout = dsel;
    out_bytes = num_pairs;
  }
  CK_LAUNCH(fn);
  if (mem == GVOX_HOST) {
    CK(cudaMemcpyAsync(counts ? (void*)counts : (void*)selected, dout, out_bytes,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return GVOX_OK;
}

}  // namespace

gvox_status gvox_overlap(gvox_ctx* ctx, const gvox_cloud* const* clouds, int64_t num_clouds,
                         const gvox_map* const* maps, int64_t num_maps, const gvox_pair* pairs,
                         int64_t num_pairs, const double* poses, int64_t num_poses, int level,
                         int32_t* counts, int mem) {
  if (!counts && num_pairs > 0) return fail(GVOX_ERR_INVALID, "gvox_overlap: counts is NULL");
  return overlap_impl("gvox_overlap", ctx, clouds, num_clouds, maps, num_maps, pairs, num_pairs,
                      poses, num_poses, level, counts, nullptr, 0, 1, mem);
}

gvox_status gvox_overlap_select(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                int64_t num_clouds, const gvox_map* const* maps, int64_t num_maps,
                                const gvox_pair* pairs, int64_t num_pairs, const double* poses,
                                int64_t num_poses, int level, int32_t num, int32_t den,
                                uint8_t* selected, int mem) {
  if (!selected && num_pairs > 0)
    return fail(GVOX_ERR_INVALID, "gvox_overlap_select: selected is NULL");
  return overlap_impl("gvox_overlap_select", ctx, clouds, num_clouds, maps, num_maps, pairs,
                      num_pairs, poses, num_poses, level, nullptr, selected, num, den, mem);
}

// ------------------------------------------------------------------ linearize
namespace {

gvox_status validate_factors(const char* fn, const gvox_cloud* const* clouds, int64_t num_clouds,
                             const gvox_map* const* maps, int64_t num_maps,
                             const gvox_factor* factors, int64_t num_factors, const double* poses,
                             int64_t num_poses) {
  for (int64_t f = 0; f < num_factors; ++f) {
    const gvox_factor& q = factors[f];
    if (clouds) {
      if (q.source_cloud < 0 || q.source_cloud >= num_clouds || !clouds[q.source_cloud])
        return fail(GVOX_ERR_INVALID, "%s: factor %lld: source_cloud %d out of range [0, %lld)", fn,
                    (long long)f, q.source_cloud, (long long)num_clouds);
    }
    if (maps) {
      if (q.target_map < 0 || q.target_map >= num_maps || !maps[q.target_map])
        return fail(GVOX_ERR_INVALID, "%s: factor %lld: target_map %d out of range [0, %lld)", fn,
                    (long long)f, q.target_map, (long long)num_maps);
    }
    if (q.pose_i < 0 || q.pose_i >= num_poses)
      return fail(GVOX_ERR_INVALID, "%s: factor %lld: pose_i %d missing (pose table has %lld)", fn,
                  (long long)f, q.pose_i, (long long)num_poses);
    if (q.pose_j < 0 || q.pose_j >= num_poses)
      return fail(GVOX_ERR_INVALID, "%s: factor %lld: pose_j %d missing (pose table has %lld)", fn,
                  (long long)f, q.pose_j, (long long)num_poses);
    if (q.flags & ~(uint32_t)(GVOX_F_VALIDATE_SURFACE | GVOX_F_ERROR_ONLY))
      return fail(GVOX_ERR_INVALID, "%s: factor %lld: unknown flags 0x%x", fn, (long long)f, q.flags);
  }
  for (int64_t i = 0; i < num_poses; ++i)
    if (!finite_pose(poses + 12 * i))
      return fail(GVOX_ERR_INVALID, "%s: pose %lld is not finite", fn, (long long)i);
  return GVOX_OK;
}

// Tile plan of a linearization batch: tiles of tile_pts consecutive points of
// one factor; tile_pts = 256 * ppt, ppt = pow2 <= n / 2048 in [1, 128] (a
// function of the factor alone: bitwise batch/shard independence).
// per-factor kernel-class bits (gvox_linearize_batch_accum_select: reduced over
// the SELECTED candidates on the device); levels in the high nibble
constexpr uint8_t kClsHash = 1, kClsNotFast = 2, kClsValidate = 4;

struct LinPlan {
  std::vector<int32_t> tstart;
  std::vector<FactorDev> fdev;
  int max_levels = 1;
  bool all_dense = true;
  bool fast = true;       // the specialised kernel: exactly 3 dyadic dense levels, no dump
  bool validate = false;  // some factor has GVOX_F_VALIDATE_SURFACE (FAST: the VALID variant)
};

gvox_status plan_linearize(const char* fn, const gvox_cloud* const* clouds,
                           const gvox_map* const* maps, const gvox_factor* factors,
                           int64_t num_factors, bool fast_allowed, LinPlan* p,
                           int min_tiles = GVOX_TILE_MIN_TILES, uint8_t* cls = nullptr) {
  p->fast = fast_allowed;
  p->tstart.assign(num_factors + 1, 0);
  p->fdev.resize(num_factors);
  int64_t corr_off = 0;
  for (int64_t f = 0; f < num_factors; ++f) {
    const gvox_factor& q = factors[f];
    const gvox_map* m = maps[q.target_map];
    if (cls) {  // this factor's kernel class alone (the screened batch decides on the device)
      bool dense = true;
      for (int l = 0; l < m->levels; ++l) dense = dense && m->desc.lv[l].dense;
      cls[f] = (uint8_t)((dense ? 0 : kClsHash) | (m->levels == 3 && m->desc.dyadic ? 0 : kClsNotFast) |
                         ((q.flags & GVOX_F_VALIDATE_SURFACE) ? kClsValidate : 0) | (m->levels << 4));
    }
    p->max_levels = std::max(p->max_levels, m->levels);
    for (int l = 0; l < m->levels; ++l) p->all_dense = p->all_dense && m->desc.lv[l].dense;
    p->fast = p->fast && m->levels == 3 && m->desc.dyadic;
    p->validate = p->validate || (q.flags & GVOX_F_VALIDATE_SURFACE);
    const int64_t n = clouds[q.source_cloud]->n;
    const int mt = n < GVOX_TILE_SMALL_N ? std::max(min_tiles, GVOX_TILE_MIN_TILES_SMALL) : min_tiles;
    int ppt = 1;
    while (ppt < GVOX_TILE_MAX_PPT && (int64_t)256 * mt * (ppt * 2) <= n) ppt *= 2;
    const int tile_pts = 256 * ppt;
    const int64_t nt = (n + tile_pts - 1) / tile_pts;
    if ((int64_t)p->tstart[f] + nt > INT32_MAX)
      return fail(GVOX_ERR_INVALID, "%s: batch too large (more than 2^31 tiles)", fn);
    p->tstart[f + 1] = p->tstart[f] + (int32_t)nt;
    FactorDev& d = p->fdev[f];
    d.src = q.source_cloud;
    d.tgt = q.target_map;
    d.pi = q.pose_i;
    d.pj = q.pose_j;
    d.flags = q.flags;
    d.tile_pts = tile_pts;
    d.corr_offset = corr_off;
    corr_off += n * m->levels;
  }
  return GVOX_OK;
}

gvox_status linearize_impl(gvox_ctx* ctx, const gvox_cloud* const* clouds, int64_t num_clouds,
                           const gvox_map* const* maps, int64_t num_maps,
                           const gvox_factor* factors, int64_t num_factors, const double* poses,
                           int64_t num_poses, gvox_linear_factor* out_full,
                           gvox_factor_accum* out_accum, int mem, int64_t* corr_dump) {
  const char* fn = out_full ? "gvox_linearize_batch" : "gvox_linearize_batch_accum";
  if (!ctx) return fail(GVOX_ERR_INVALID, "%s: ctx is NULL", fn);
  if (num_factors < 0) return fail(GVOX_ERR_INVALID, "%s: num_factors < 0", fn);
  if (num_factors == 0) return GVOX_OK;
  if (!clouds || !maps || !factors || !poses || !(out_full || out_accum))
    return fail(GVOX_ERR_INVALID, "%s: NULL argument", fn);
  if (mem != GVOX_HOST && mem != GVOX_DEVICE)
    return fail(GVOX_ERR_INVALID, "%s: mem must be GVOX_HOST or GVOX_DEVICE", fn);
  gvox_status st = validate_factors(fn, clouds, num_clouds, maps, num_maps, factors, num_factors,
                                    poses, num_poses);
  if (st) return st;
  DeviceGuard g(ctx->device);
  LinPlan plan;
  st = plan_linearize(fn, clouds, maps, factors, num_factors,
                      corr_dump == nullptr && std::getenv("GVOX_LIN_GENERIC") == nullptr, &plan);
  if (st) return st;
  const std::vector<int32_t>& tstart = plan.tstart;
  const std::vector<FactorDev>& fdev = plan.fdev;
  const int max_levels = plan.max_levels;
  const bool all_dense = plan.all_dense, fast = plan.fast;
  const int64_t T = tstart[num_factors];
  // ---- the single serialized input block
  Layout lay;
  size_t o_pose = lay.add(96 * num_poses);
  size_t o_fac = lay.add(sizeof(FactorDev) * num_factors);
  size_t o_ts = lay.add(4 * (num_factors + 1));
  const bool host_tm = T <= kHostTileMapMax;
  size_t o_tm = lay.add(host_tm ? 4 * (size_t)T : 0);
  // large batches: tiles executed grouped by target map (host counting sort)
  const bool by_target = exec_by_target() && T > kHostTileMapMax && num_factors > 1;
  size_t o_ex = lay.add(by_target ? 4 * (size_t)T : 0);
  size_t o_cl = lay.add(8 * num_clouds);
  size_t o_mp = lay.add(8 * num_maps);
  const size_t in_bytes = lay.size;
  void* pin = nullptr;
  st = pin_reserve(ctx, in_bytes, &pin);
  if (st) return st;
  char* hp = (char*)pin;
  std::memcpy(hp + o_pose, poses, 96 * num_poses);
  std::memcpy(hp + o_fac, fdev.data(), sizeof(FactorDev) * num_factors);
  std::memcpy(hp + o_ts, tstart.data(), 4 * (num_factors + 1));
  if (host_tm) fill_tile_map(tstart.data(), num_factors, (int32_t*)(hp + o_tm));
  if (by_target) {
    std::vector<int32_t> cur((size_t)num_maps + 1, 0);
    for (int64_t f = 0; f < num_factors; ++f) cur[fdev[f].tgt + 1] += tstart[f + 1] - tstart[f];
    for (int64_t m = 0; m < num_maps; ++m) cur[m + 1] += cur[m];
    int32_t* ex = (int32_t*)(hp + o_ex);
    for (int64_t f = 0; f < num_factors; ++f)
      for (int32_t t = tstart[f]; t < tstart[f + 1]; ++t) ex[cur[fdev[f].tgt]++] = t;
  }
  for (int64_t i = 0; i < num_clouds; ++i) ((const CloudDev**)(hp + o_cl))[i] = clouds[i] ? clouds[i]->dev : nullptr;
  for (int64_t i = 0; i < num_maps; ++i) ((const MapDev**)(hp + o_mp))[i] = maps[i] ? maps[i]->dev : nullptr;
  // ---- device workspace
  Layout wl;
  size_t o_in = wl.add(in_bytes);
  size_t o_part = wl.add(8 * kPartialStride * (size_t)std::max<int64_t>(T, 1));
  size_t o_tf = wl.add(host_tm ? 0 : 4 * (size_t)std::max<int64_t>(T, 1));
  size_t out_rec = out_full ? sizeof(gvox_linear_factor) : sizeof(gvox_factor_accum);
  size_t o_out = wl.add(mem == GVOX_HOST ? out_rec * num_factors : 0);
  void* ws = nullptr;
  st = ws_reserve(ctx, 0, wl.size, &ws);
  if (st) return st;
  char* wb = (char*)ws;
  st = h2d_block(ctx, wb + o_in, hp, in_bytes);
  if (st) return st;
  char* din = wb + o_in;
  void* dout = mem == GVOX_DEVICE ? (out_full ? (void*)out_full : (void*)out_accum) : (void*)(wb + o_out);
  int32_t* dtf = host_tm ? (int32_t*)(din + o_tm) : (int32_t*)(wb + o_tf);
  if (!host_tm) launch_tile_map((const int32_t*)(din + o_ts), num_factors, dtf, ctx->stream);
  {
    TimerScope ts(ctx, GVOX_TIMER_LINEARIZE);
    launch_linearize((const CloudDev* const*)(din + o_cl), (const MapDev* const*)(din + o_mp),
                     (const FactorDev*)(din + o_fac), (const int32_t*)(din + o_ts), num_factors, T,
                     0, max_levels, (const double*)(din + o_pose), (double*)(wb + o_part),
                     dtf, corr_dump, all_dense, fast, plan.validate,
                     ctx->stream, by_target ? (const int32_t*)(din + o_ex) : nullptr);
  }
  CK_LAUNCH("linearize");
  {
    TimerScope ts(ctx, GVOX_TIMER_REDUCE);
    launch_reduce((const FactorDev*)(din + o_fac), (const int32_t*)(din + o_ts), num_factors,
                  (const double*)(din + o_pose), (const double*)(wb + o_part),
                  out_full ? (gvox_linear_factor*)dout : nullptr,
                  out_full ? nullptr : (gvox_factor_accum*)dout, ctx->stream);
  }
  CK_LAUNCH("linearize reduce");
  if (mem == GVOX_HOST) {
    void* host_out = out_full ? (void*)out_full : (void*)out_accum;
    CK(cudaMemcpyAsync(host_out, dout, out_rec * num_factors, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return GVOX_OK;
}

}  // namespace

gvox_status gvox_linearize_batch(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                 int64_t num_clouds, const gvox_map* const* maps, int64_t num_maps,
                                 const gvox_factor* factors, int64_t num_factors,
                                 const double* poses, int64_t num_poses, gvox_linear_factor* out,
                                 int mem, int64_t* corr_dump) {
  if (!out && num_factors > 0) return fail(GVOX_ERR_INVALID, "gvox_linearize_batch: out is NULL");
  return linearize_impl(ctx, clouds, num_clouds, maps, num_maps, factors, num_factors, poses,
                        num_poses, out, nullptr, mem, corr_dump);
}

gvox_status gvox_linearize_batch_accum(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                       int64_t num_clouds, const gvox_map* const* maps,
                                       int64_t num_maps, const gvox_factor* factors,
                                       int64_t num_factors, const double* poses, int64_t num_poses,
                                       gvox_factor_accum* out, int mem) {
  if (!out && num_factors > 0) return fail(GVOX_ERR_INVALID, "gvox_linearize_batch_accum: out is NULL");
  return linearize_impl(ctx, clouds, num_clouds, maps, num_maps, factors, num_factors, poses,
                        num_poses, nullptr, out, mem, nullptr);
}

gvox_status gvox_linearize_batch_accum_select(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                              int64_t num_clouds, const gvox_map* const* maps,
                                              int64_t num_maps, const gvox_factor* candidates,
                                              int64_t num_candidates, const uint8_t* selected,
                                              const double* poses, int64_t num_poses,
                                              gvox_factor_accum* out, int64_t* num_selected,
                                              uint8_t* selected_host) {
  const char* fn = "gvox_linearize_batch_accum_select";
  if (!ctx) return fail(GVOX_ERR_INVALID, "%s: ctx is NULL", fn);
  if (num_candidates < 0) return fail(GVOX_ERR_INVALID, "%s: num_candidates < 0", fn);
  if (!num_selected) return fail(GVOX_ERR_INVALID, "%s: num_selected is NULL", fn);
  *num_selected = 0;
  if (num_candidates == 0) return GVOX_OK;
  if (!clouds || !maps || !candidates || !selected || !poses || !out)
    return fail(GVOX_ERR_INVALID, "%s: NULL argument", fn);
  if (num_candidates > INT32_MAX) return fail(GVOX_ERR_INVALID, "%s: more than 2^31 candidates", fn);
  gvox_status st = validate_factors(fn, clouds, num_clouds, maps, num_maps, candidates,
                                    num_candidates, poses, num_poses);
  if (st) return st;
  DeviceGuard g(ctx->device);
  // host plan of every candidate (tiles are a function of the factor alone, so
  // the selected subset's tiles are exactly gvox_linearize_batch_accum's)
  LinPlan plan;
  std::vector<uint8_t> cls(num_candidates);
  st = plan_linearize(fn, clouds, maps, candidates, num_candidates,
                      std::getenv("GVOX_LIN_GENERIC") == nullptr, &plan, GVOX_TILE_MIN_TILES,
                      cls.data());
  if (st) return st;
  const int64_t T_all = plan.tstart[num_candidates];
  std::vector<int32_t> ntiles(num_candidates);
  for (int64_t p = 0; p < num_candidates; ++p) ntiles[p] = plan.tstart[p + 1] - plan.tstart[p];
  // ---- the single serialized input block
  Layout lay;
  size_t o_pose = lay.add(96 * num_poses);
  size_t o_fac = lay.add(sizeof(FactorDev) * num_candidates);
  size_t o_nt = lay.add(4 * num_candidates);
  size_t o_cls = lay.add(num_candidates);
  size_t o_cl = lay.add(8 * num_clouds);
  size_t o_mp = lay.add(8 * num_maps);
  const size_t in_bytes = lay.size;
  void* pin = nullptr;
  st = pin_reserve(ctx, in_bytes, &pin);
  if (st) return st;
  char* hp = (char*)pin;
  std::memcpy(hp + o_pose, poses, 96 * num_poses);
  std::memcpy(hp + o_fac, plan.fdev.data(), sizeof(FactorDev) * num_candidates);
  std::memcpy(hp + o_nt, ntiles.data(), 4 * num_candidates);
  std::memcpy(hp + o_cls, cls.data(), num_candidates);
  for (int64_t i = 0; i < num_clouds; ++i) ((const CloudDev**)(hp + o_cl))[i] = clouds[i] ? clouds[i]->dev : nullptr;
  for (int64_t i = 0; i < num_maps; ++i) ((const MapDev**)(hp + o_mp))[i] = maps[i] ? maps[i]->dev : nullptr;
  // ---- device workspace (partials and tile map sized for every candidate)
  Layout wl;
  size_t o_in = wl.add(in_bytes);
  size_t o_part = wl.add(8 * kPartialStride * (size_t)std::max<int64_t>(T_all, 1));
  size_t o_tf = wl.add(4 * (size_t)std::max<int64_t>(T_all, 1));
  size_t o_fc = wl.add(sizeof(FactorDev) * num_candidates);
  size_t o_tsc = wl.add(4 * (num_candidates + 1));
  size_t o_cnt = wl.add(16);
  // tiles grouped by target map for execution (GVOX_LIN_EXEC_ORDER=0: batch order)
  const bool by_target = exec_by_target();
  size_t o_hist = wl.add(by_target ? 4 * (size_t)std::max<int64_t>(num_maps, 1) : 0);
  size_t o_exec = wl.add(by_target ? 4 * (size_t)std::max<int64_t>(T_all, 1) : 0);
  size_t o_bt = wl.add(8 * ((num_candidates + 1023) / 1024));
  void* ws = nullptr;
  st = ws_reserve(ctx, 0, wl.size, &ws);
  if (st) return st;
  char* wb = (char*)ws;
  st = h2d_block(ctx, wb + o_in, hp, in_bytes);
  if (st) return st;
  char* din = wb + o_in;
  FactorDev* fc = (FactorDev*)(wb + o_fc);
  int32_t* tsc = (int32_t*)(wb + o_tsc);
  int32_t* dcnt = (int32_t*)(wb + o_cnt);
  launch_select_plan(selected, (const int32_t*)(din + o_nt), (const uint8_t*)(din + o_cls),
                     (const FactorDev*)(din + o_fac), num_candidates, fc, tsc, dcnt,
                     (int2*)(wb + o_bt), ctx->stream);
  CK_LAUNCH("select plan");
  // the one readback before the launch: {S, T} (the grid size) and the kernel
  // class of the selected candidates {OR of their class bits, max levels}
  if (!ctx->pin_counts) {
    cudaError_t e = cudaHostAlloc((void**)&ctx->pin_counts, 64, cudaHostAllocDefault);
    if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc");
  }
  CK(cudaMemcpyAsync(ctx->pin_counts, dcnt, 16, cudaMemcpyDeviceToHost, ctx->stream));
  if (selected_host)
    CK(cudaMemcpyAsync(selected_host, selected, num_candidates, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const int64_t S = ctx->pin_counts[0], T = ctx->pin_counts[1];
  const int32_t cls_or = ctx->pin_counts[2], sel_levels = ctx->pin_counts[3];
  *num_selected = S;
  if (S == 0) return GVOX_OK;
  // the kernel variant of the SELECTED batch (as gvox_linearize_batch_accum would
  // choose it on that list), not of every candidate
  plan.fast = std::getenv("GVOX_LIN_GENERIC") == nullptr && !(cls_or & kClsNotFast);
  plan.all_dense = !(cls_or & kClsHash);
  plan.validate = (cls_or & kClsValidate) != 0;
  plan.max_levels = std::max(1, sel_levels);
  launch_tile_map(tsc, S, (int32_t*)(wb + o_tf), ctx->stream);
  if (by_target)
    launch_exec_order_by_target(fc, tsc, S, num_maps, (int32_t*)(wb + o_hist), (int32_t*)(wb + o_exec),
                                ctx->stream);
  {
    TimerScope ts(ctx, GVOX_TIMER_LINEARIZE);
    launch_linearize((const CloudDev* const*)(din + o_cl), (const MapDev* const*)(din + o_mp), fc,
                     tsc, S, T, 0, plan.max_levels, (const double*)(din + o_pose),
                     (double*)(wb + o_part), (int32_t*)(wb + o_tf), nullptr, plan.all_dense,
                     plan.fast, plan.validate, ctx->stream,
                     by_target ? (const int32_t*)(wb + o_exec) : nullptr);
  }
  CK_LAUNCH("linearize");
  {
    TimerScope ts(ctx, GVOX_TIMER_REDUCE);
    launch_reduce(fc, tsc, S, (const double*)(din + o_pose), (const double*)(wb + o_part), nullptr,
                  out, ctx->stream);
  }
  CK_LAUNCH("linearize reduce");
  return GVOX_OK;
}

gvox_status gvox_expand(gvox_ctx* ctx, const gvox_factor* factors, int64_t num_factors,
                        const double* poses, int64_t num_poses, const gvox_factor_accum* accum,
                        gvox_linear_factor* out, int mem) {
  if (!ctx) return fail(GVOX_ERR_INVALID, "gvox_expand: ctx is NULL");
  if (num_factors < 0) return fail(GVOX_ERR_INVALID, "gvox_expand: num_factors < 0");
  if (num_factors == 0) return GVOX_OK;
  if (!factors || !poses || !accum || !out) return fail(GVOX_ERR_INVALID, "gvox_expand: NULL argument");
  gvox_status st = validate_factors("gvox_expand", nullptr, 0, nullptr, 0, factors, num_factors,
                                    poses, num_poses);
  if (st) return st;
  DeviceGuard g(ctx->device);
  std::vector<FactorDev> fdev(num_factors);
  for (int64_t f = 0; f < num_factors; ++f) {
    fdev[f] = FactorDev{factors[f].source_cloud, factors[f].target_map, factors[f].pose_i,
                        factors[f].pose_j, factors[f].flags, 0, 0};  // tiles unused by expand
  }
  Layout lay;
  size_t o_pose = lay.add(96 * num_poses);
  size_t o_fac = lay.add(sizeof(FactorDev) * num_factors);
  void* pin = nullptr;
  st = pin_reserve(ctx, lay.size, &pin);
  if (st) return st;
  std::memcpy((char*)pin + o_pose, poses, 96 * num_poses);
  std::memcpy((char*)pin + o_fac, fdev.data(), sizeof(FactorDev) * num_factors);
  Layout wl;
  size_t o_in = wl.add(lay.size);
  size_t o_out = wl.add(mem == GVOX_HOST ? sizeof(gvox_linear_factor) * num_factors : 0);
  void* ws = nullptr;
  st = ws_reserve(ctx, 0, wl.size, &ws);
  if (st) return st;
  char* wb = (char*)ws;
  st = h2d_block(ctx, wb + o_in, pin, lay.size);
  if (st) return st;
  gvox_linear_factor* dout = mem == GVOX_DEVICE ? out : (gvox_linear_factor*)(wb + o_out);
  launch_expand((const FactorDev*)(wb + o_in + o_fac), num_factors,
                (const double*)(wb + o_in + o_pose), accum, dout, ctx->stream);
  CK_LAUNCH("gvox_expand");
  if (mem == GVOX_HOST) {
    CK(cudaMemcpyAsync(out, dout, sizeof(gvox_linear_factor) * num_factors,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return GVOX_OK;
}

// ------------------------------------------------------------ preprocessing
namespace {

// common validation + point upload + per-cloud tile plan for the
// preprocessing calls
struct PrepBatch {
  const float* dpts = nullptr;          // device points
  std::vector<KnnCloudDev> cl;
  std::vector<int32_t> tstart;
  int tile_pts = 64;  // one query per thread (64-thread CTAs): a single frame spreads over all SMs
  int64_t n = 0, T = 0;
};

gvox_status prep_batch(const char* fn, gvox_ctx* ctx, const float* points, const int64_t* offsets,
                       int64_t count, int mem, void* dev_points_ws, PrepBatch* b) {
  if (count < 0) return fail(GVOX_ERR_INVALID, "%s: count < 0", fn);
  if (!offsets) return fail(GVOX_ERR_INVALID, "%s: offsets is NULL", fn);
  if (offsets[0] != 0) return fail(GVOX_ERR_INVALID, "%s: offsets[0] != 0", fn);
  for (int64_t c = 0; c < count; ++c)
    if (offsets[c + 1] < offsets[c])
      return fail(GVOX_ERR_INVALID, "%s: offsets not non-decreasing at cloud %lld", fn, (long long)c);
  b->n = offsets[count];
  if (b->n > INT32_MAX) return fail(GVOX_ERR_INVALID, "%s: more than 2^31 points", fn);
  if (b->n > 0 && !points) return fail(GVOX_ERR_INVALID, "%s: points is NULL", fn);
  b->cl.resize(count);
  b->tstart.assign(count + 1, 0);
  for (int64_t c = 0; c < count; ++c) {
    KnnCloudDev& d = b->cl[c];
    std::memset(&d, 0, sizeof(d));
    d.first = offsets[c];
    d.n = offsets[c + 1] - offsets[c];
    b->tstart[c + 1] = b->tstart[c] + (int32_t)((d.n + b->tile_pts - 1) / b->tile_pts);
  }
  b->T = b->tstart[count];
  if (mem == GVOX_DEVICE || b->n == 0) {
    b->dpts = points;
  } else {
    CK(cudaMemcpyAsync(dev_points_ws, points, 12 * b->n, cudaMemcpyHostToDevice, ctx->stream));
    b->dpts = (const float*)dev_points_ws;
  }
  return GVOX_OK;
}

}  // namespace

gvox_status gvox_knn(gvox_ctx* ctx, const float* points, const int64_t* offsets, int64_t count,
                     int32_t k, double cell_size, int32_t* neighbors, int mem) {
  const char* fn = "gvox_knn";
  if (!ctx) return fail(GVOX_ERR_INVALID, "%s: ctx is NULL", fn);
  if (k < 1 || k > 32) return fail(GVOX_ERR_INVALID, "%s: k = %d outside [1, 32]", fn, k);
  if (!(cell_size > 0.0) || !std::isfinite(cell_size))
    return fail(GVOX_ERR_INVALID, "%s: cell_size must be finite and > 0", fn);
  if (mem != GVOX_HOST && mem != GVOX_DEVICE)
    return fail(GVOX_ERR_INVALID, "%s: mem must be GVOX_HOST or GVOX_DEVICE", fn);
  if (count < 0 || !offsets) return fail(GVOX_ERR_INVALID, "%s: bad count / offsets", fn);
  const int64_t n_all = count > 0 ? offsets[count] : 0;
  if (n_all > 0 && !neighbors) return fail(GVOX_ERR_INVALID, "%s: neighbors is NULL", fn);
  DeviceGuard g(ctx->device);
  // workspace 1: uploaded points (host input), bbox, the cloud / tile tables
  void* ws1 = nullptr;
  Layout l1;
  size_t o_pts = l1.add(mem == GVOX_HOST ? 12 * (size_t)std::max<int64_t>(n_all, 0) : 0);
  size_t o_box = l1.add(4 * 6 * (size_t)std::max<int64_t>(count, 1) + 16);
  size_t o_cl = l1.add(sizeof(KnnCloudDev) * (size_t)std::max<int64_t>(count, 1));
  size_t o_ts = l1.add(4 * (size_t)(count + 1));
  size_t o_tc = l1.add(4 * (size_t)(n_all / 64 + count + 1));
  gvox_status st = ws_reserve(ctx, 1, l1.size, &ws1);
  if (st) return st;
  char* w1 = (char*)ws1;
  PrepBatch b;
  st = prep_batch(fn, ctx, points, offsets, count, mem, w1 + o_pts, &b);
  if (st) return st;
  if (b.n == 0) return GVOX_OK;
  // ---- bounding boxes (one sync: the grids are sized on the host)
  {
    void* pin = nullptr;
    Layout lp;
    size_t p_cl = lp.add(sizeof(KnnCloudDev) * count);
    size_t p_ts = lp.add(4 * (count + 1));
    size_t p_box = lp.add(4 * 6 * count + 16);
    st = pin_reserve(ctx, lp.size, &pin);
    if (st) return st;
    char* hp = (char*)pin;
    std::memcpy(hp + p_cl, b.cl.data(), sizeof(KnnCloudDev) * count);
    std::memcpy(hp + p_ts, b.tstart.data(), 4 * (count + 1));
    int32_t* hb = (int32_t*)(hp + p_box);
    for (int64_t c = 0; c < count; ++c)
      for (int a = 0; a < 3; ++a) {
        hb[6 * c + a] = INT32_MAX;
        hb[6 * c + 3 + a] = INT32_MIN;
      }
    hb[6 * count] = 0;  // non-finite flag
    CK(cudaMemcpyAsync(w1 + o_cl, hp + p_cl, sizeof(KnnCloudDev) * count, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(w1 + o_ts, hp + p_ts, 4 * (count + 1), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(w1 + o_box, hp + p_box, 4 * (6 * count + 1), cudaMemcpyHostToDevice, ctx->stream));
    launch_tile_map((const int32_t*)(w1 + o_ts), count, (int32_t*)(w1 + o_tc), ctx->stream);
    launch_knn_bbox(b.dpts, (const KnnCloudDev*)(w1 + o_cl), (const int32_t*)(w1 + o_ts),
                    (const int32_t*)(w1 + o_tc), b.T, b.tile_pts, (int32_t*)(w1 + o_box),
                    (int32_t*)(w1 + o_box) + 6 * count, ctx->stream);
    CK_LAUNCH(fn);
    CK(cudaMemcpyAsync(hb, w1 + o_box, 4 * (6 * count + 1), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->pin_ring[ctx->pin_slot].pending = false;
    if (hb[6 * count]) return fail(GVOX_ERR_INVALID, "%s: non-finite point coordinate", fn);
    if (std::getenv("GVOX_DEBUG_KNN"))
      for (int64_t c = 0; c < count; ++c)
        fprintf(stderr, "[gvox_knn] cloud %lld n %lld box %g %g %g .. %g %g %g (mem %d, pts %p)\n",
                (long long)c, (long long)b.cl[c].n, ordered_to_float(hb[6 * c]),
                ordered_to_float(hb[6 * c + 1]), ordered_to_float(hb[6 * c + 2]),
                ordered_to_float(hb[6 * c + 3]), ordered_to_float(hb[6 * c + 4]),
                ordered_to_float(hb[6 * c + 5]), mem, (const void*)b.dpts);
    // ---- per-cloud grids: pitch cell_size, doubled while the grid would
    // hold more than 32 cells per point (sparse extents)
    int64_t cells = 0;
    for (int64_t c = 0; c < count; ++c) {
      KnnCloudDev& d = b.cl[c];
      if (d.n == 0) {
        d.s = cell_size;
        d.inv_s = 1.0 / cell_size;
        d.dim[0] = d.dim[1] = d.dim[2] = 1;
        d.cell0 = (int32_t)cells;
        cells += 1;
        continue;
      }
      double lo[3], hi[3];
      for (int a = 0; a < 3; ++a) {
        lo[a] = ordered_to_float(hb[6 * c + a]);
        hi[a] = ordered_to_float(hb[6 * c + 3 + a]);
        if (!(hi[a] >= lo[a]) || !std::isfinite(hi[a] - lo[a]))
          return fail(GVOX_ERR_INVALID, "%s: cloud %lld: bad bounding box [%g, %g] on axis %d", fn,
                      (long long)c, lo[a], hi[a], a);
      }
      double s = cell_size;
      int64_t dims[3], nc;
      for (;;) {
        nc = 1;
        for (int a = 0; a < 3; ++a) {
          dims[a] = (int64_t)std::floor((hi[a] - lo[a]) / s) + 1;
          nc *= dims[a];
        }
        if (nc <= std::max<int64_t>(32 * d.n, 4096) && nc < (1ll << 30)) break;
        s *= 2.0;
      }
      for (int a = 0; a < 3; ++a) {
        d.lo[a] = lo[a];
        d.dim[a] = (int32_t)dims[a];
      }
      d.s = s;
      d.inv_s = 1.0 / s;
      d.cell0 = (int32_t)cells;
      cells += nc;
      if (cells >= INT32_MAX) return fail(GVOX_ERR_INVALID, "%s: search grids exceed 2^31 cells", fn);
    }
    CK(cudaMemcpyAsync(w1 + o_cl, b.cl.data(), sizeof(KnnCloudDev) * count, cudaMemcpyHostToDevice,
                       ctx->stream));
    // (pageable copy of a host vector: synchronous with respect to the host)
    Layout l2;
    size_t o_cnt = l2.add(4 * (size_t)(cells + 1));
    size_t o_start = l2.add(4 * (size_t)(cells + 1));
    size_t o_fill = l2.add(4 * (size_t)(cells + 1));
    size_t o_scr = l2.add(4 * (size_t)(cells / 4096 + 2));
    size_t o_cell = l2.add(4 * (size_t)b.n);
    size_t o_sorted = l2.add(16 * (size_t)b.n);
    size_t o_out = l2.add(mem == GVOX_HOST ? 4 * (size_t)b.n * k : 0);
    void* ws2 = nullptr;
    st = ws_reserve(ctx, 2, l2.size, &ws2);
    if (st) return st;
    char* w2 = (char*)ws2;
    CK(cudaMemsetAsync(w2 + o_cnt, 0, 4 * (size_t)(cells + 1), ctx->stream));
    CK(cudaMemsetAsync(w2 + o_fill, 0, 4 * (size_t)(cells + 1), ctx->stream));
    const KnnCloudDev* dcl = (const KnnCloudDev*)(w1 + o_cl);
    const int32_t* dts = (const int32_t*)(w1 + o_ts);
    const int32_t* dtc = (const int32_t*)(w1 + o_tc);
    int32_t* dout = mem == GVOX_DEVICE ? neighbors : (int32_t*)(w2 + o_out);
    TimerScope ts(ctx, GVOX_TIMER_PREPROCESS);
    launch_knn_count(b.dpts, dcl, dts, dtc, b.T, b.tile_pts, (int32_t*)(w2 + o_cell),
                     (int32_t*)(w2 + o_cnt), ctx->stream);
    launch_exclusive_scan((const int32_t*)(w2 + o_cnt), cells, (int32_t*)(w2 + o_start),
                          (int32_t*)(w2 + o_scr), ctx->stream);
    launch_knn_scatter(b.dpts, dcl, dts, dtc, b.T, b.tile_pts, (const int32_t*)(w2 + o_cell),
                       (const int32_t*)(w2 + o_start), (int32_t*)(w2 + o_fill),
                       (float4*)(w2 + o_sorted), ctx->stream);
    launch_knn_query(dcl, dts, dtc, b.T, b.tile_pts, (const float4*)(w2 + o_sorted),
                     (const int32_t*)(w2 + o_start), k, dout, ctx->stream);
    CK_LAUNCH(fn);
    if (mem == GVOX_HOST) {
      CK(cudaMemcpyAsync(neighbors, dout, 4 * (size_t)b.n * k, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    }
  }
  return GVOX_OK;
}

gvox_status gvox_estimate_covariances(gvox_ctx* ctx, const float* points, const int64_t* offsets,
                                      int64_t count, const int32_t* neighbors, int32_t k,
                                      float* cov, float* normals, int mem) {
  const char* fn = "gvox_estimate_covariances";
  if (!ctx) return fail(GVOX_ERR_INVALID, "%s: ctx is NULL", fn);
  if (k < 1 || k > 32) return fail(GVOX_ERR_INVALID, "%s: k = %d outside [1, 32]", fn, k);
  if (mem != GVOX_HOST && mem != GVOX_DEVICE)
    return fail(GVOX_ERR_INVALID, "%s: mem must be GVOX_HOST or GVOX_DEVICE", fn);
  if (count < 0 || !offsets) return fail(GVOX_ERR_INVALID, "%s: bad count / offsets", fn);
  const int64_t n_all = count > 0 ? offsets[count] : 0;
  if (n_all > 0 && (!neighbors || !cov || !normals)) return fail(GVOX_ERR_INVALID, "%s: NULL argument", fn);
  if (mem == GVOX_HOST)
    for (int64_t c = 0; c < count; ++c)
      for (int64_t i = offsets[c]; i < offsets[c + 1]; ++i)
        for (int j = 0; j < k; ++j) {
          const int32_t q = neighbors[i * k + j];
          if (q < -1 || q >= offsets[c + 1] - offsets[c])
            return fail(GVOX_ERR_INVALID, "%s: neighbors[%lld][%d] = %d outside [-1, %lld)", fn,
                        (long long)i, j, q, (long long)(offsets[c + 1] - offsets[c]));
        }
  DeviceGuard g(ctx->device);
  Layout l1;
  size_t o_pts = l1.add(mem == GVOX_HOST ? 12 * (size_t)n_all : 0);
  size_t o_nb = l1.add(mem == GVOX_HOST ? 4 * (size_t)n_all * k : 0);
  size_t o_cov = l1.add(mem == GVOX_HOST ? 24 * (size_t)n_all : 0);
  size_t o_nrm = l1.add(mem == GVOX_HOST ? 12 * (size_t)n_all : 0);
  size_t o_cl = l1.add(sizeof(KnnCloudDev) * (size_t)std::max<int64_t>(count, 1));
  size_t o_ts = l1.add(4 * (size_t)(count + 1));
  size_t o_tc = l1.add(4 * (size_t)(n_all / 64 + count + 1));
  void* ws = nullptr;
  gvox_status st = ws_reserve(ctx, 1, l1.size, &ws);
  if (st) return st;
  char* w = (char*)ws;
  PrepBatch b;
  st = prep_batch(fn, ctx, points, offsets, count, mem, w + o_pts, &b);
  if (st) return st;
  if (b.n == 0) return GVOX_OK;
  const int32_t* dnb = neighbors;
  float* dcov = cov;
  float* dnrm = normals;
  if (mem == GVOX_HOST) {
    CK(cudaMemcpyAsync(w + o_nb, neighbors, 4 * (size_t)b.n * k, cudaMemcpyHostToDevice, ctx->stream));
    dnb = (const int32_t*)(w + o_nb);
    dcov = (float*)(w + o_cov);
    dnrm = (float*)(w + o_nrm);
  }
  CK(cudaMemcpyAsync(w + o_cl, b.cl.data(), sizeof(KnnCloudDev) * count, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(w + o_ts, b.tstart.data(), 4 * (count + 1), cudaMemcpyHostToDevice, ctx->stream));
  launch_tile_map((const int32_t*)(w + o_ts), count, (int32_t*)(w + o_tc), ctx->stream);
  {
    TimerScope ts(ctx, GVOX_TIMER_PREPROCESS);
    launch_covariance(b.dpts, (const KnnCloudDev*)(w + o_cl), (const int32_t*)(w + o_ts),
                      (const int32_t*)(w + o_tc), b.T, b.tile_pts, dnb, k, dcov, dnrm, ctx->stream);
  }
  CK_LAUNCH(fn);
  if (mem == GVOX_HOST) {
    CK(cudaMemcpyAsync(cov, dcov, 24 * (size_t)b.n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(normals, dnrm, 12 * (size_t)b.n, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return GVOX_OK;
}

// ------------------------------------------------------------ keyframes
gvox_status gvox_overlap_union(gvox_ctx* ctx, const gvox_cloud* const* clouds, int64_t num_clouds,
                               const gvox_map* const* maps, int64_t num_maps,
                               const gvox_union_query* queries, int64_t num_queries,
                               const gvox_union_member* members, int64_t num_members,
                               const double* poses, int64_t num_poses, int level,
                               int32_t* counts, int mem) {
  const char* fn = "gvox_overlap_union";
  if (!ctx) return fail(GVOX_ERR_INVALID, "%s: ctx is NULL", fn);
  if (num_queries < 0 || num_members < 0) return fail(GVOX_ERR_INVALID, "%s: negative size", fn);
  if (num_queries == 0) return GVOX_OK;
  if (!clouds || !queries || !poses || !counts || (num_members > 0 && (!members || !maps)))
    return fail(GVOX_ERR_INVALID, "%s: NULL argument", fn);
  if (mem != GVOX_HOST && mem != GVOX_DEVICE)
    return fail(GVOX_ERR_INVALID, "%s: mem must be GVOX_HOST or GVOX_DEVICE", fn);
  if (num_queries > INT32_MAX || num_members > INT32_MAX)
    return fail(GVOX_ERR_INVALID, "%s: more than 2^31 queries or members", fn);
  for (int64_t m = 0; m < num_members; ++m) {
    const gvox_union_member& u = members[m];
    if (u.target_map < 0 || u.target_map >= num_maps || !maps[u.target_map])
      return fail(GVOX_ERR_INVALID, "%s: member %lld: target_map %d out of range [0, %lld)", fn,
                  (long long)m, u.target_map, (long long)num_maps);
    if (u.pose_j < 0 || u.pose_j >= num_poses)
      return fail(GVOX_ERR_INVALID, "%s: member %lld: pose_j %d out of range [0, %lld)", fn,
                  (long long)m, u.pose_j, (long long)num_poses);
    if (level < 0 || level >= maps[u.target_map]->levels)
      return fail(GVOX_ERR_INVALID, "%s: member %lld: level %d outside the map's [0, %d)", fn,
                  (long long)m, level, maps[u.target_map]->levels);
  }
  for (int64_t q = 0; q < num_queries; ++q) {
    const gvox_union_query& u = queries[q];
    if (u.source_cloud < 0 || u.source_cloud >= num_clouds || !clouds[u.source_cloud])
      return fail(GVOX_ERR_INVALID, "%s: query %lld: source_cloud %d out of range [0, %lld)", fn,
                  (long long)q, u.source_cloud, (long long)num_clouds);
    if (u.pose_i < 0 || u.pose_i >= num_poses)
      return fail(GVOX_ERR_INVALID, "%s: query %lld: pose_i %d out of range [0, %lld)", fn,
                  (long long)q, u.pose_i, (long long)num_poses);
    if (u.count < 0 || u.first < 0 || (int64_t)u.first + u.count > num_members)
      return fail(GVOX_ERR_INVALID, "%s: query %lld: members [%d, %d + %d) outside [0, %lld)", fn,
                  (long long)q, u.first, u.first, u.count, (long long)num_members);
  }
  for (int64_t i = 0; i < num_poses; ++i)
    if (!finite_pose(poses + 12 * i))
      return fail(GVOX_ERR_INVALID, "%s: pose %lld is not finite", fn, (long long)i);
  DeviceGuard g(ctx->device);
  // tiles of 256 * ppt points (ppt <= 32: one hit bit per point and thread)
  int64_t total = 0;
  for (int64_t q = 0; q < num_queries; ++q)
    if (queries[q].count > 0) total += clouds[queries[q].source_cloud]->n;
  int ppt = 1;
  while (ppt < 32 && total / ((int64_t)256 * ppt * 2) >= 148 * 8) ppt *= 2;
  const int tile_pts = 256 * ppt;
  std::vector<int32_t> tstart(num_queries + 1, 0);
  for (int64_t q = 0; q < num_queries; ++q) {
    const int64_t n = queries[q].count > 0 ? clouds[queries[q].source_cloud]->n : 0;
    const int64_t nt = tstart[q] + (n + tile_pts - 1) / tile_pts;
    if (nt > INT32_MAX) return fail(GVOX_ERR_INVALID, "%s: more than 2^31 tiles", fn);
    tstart[q + 1] = (int32_t)nt;
  }
  const int64_t T = tstart.back();
  Layout lay;
  size_t o_pose = lay.add(96 * num_poses);
  size_t o_q = lay.add(sizeof(UnionQueryDev) * num_queries);
  size_t o_m = lay.add(sizeof(UnionMemberDev) * std::max<int64_t>(num_members, 1));
  size_t o_ts = lay.add(4 * tstart.size());
  size_t o_cl = lay.add(8 * num_clouds);
  size_t o_mp = lay.add(8 * std::max<int64_t>(num_maps, 1));
  const size_t in_bytes = lay.size;
  void* pin = nullptr;
  gvox_status st = pin_reserve(ctx, in_bytes, &pin);
  if (st) return st;
  char* hp = (char*)pin;
  std::memcpy(hp + o_pose, poses, 96 * num_poses);
  static_assert(sizeof(UnionQueryDev) == sizeof(gvox_union_query), "layout");
  static_assert(sizeof(UnionMemberDev) == sizeof(gvox_union_member), "layout");
  std::memcpy(hp + o_q, queries, sizeof(UnionQueryDev) * num_queries);
  if (num_members) std::memcpy(hp + o_m, members, sizeof(UnionMemberDev) * num_members);
  std::memcpy(hp + o_ts, tstart.data(), 4 * tstart.size());
  for (int64_t i = 0; i < num_clouds; ++i) ((const CloudDev**)(hp + o_cl))[i] = clouds[i] ? clouds[i]->dev : nullptr;
  for (int64_t i = 0; i < num_maps; ++i) ((const MapDev**)(hp + o_mp))[i] = maps[i] ? maps[i]->dev : nullptr;
  Layout wl;
  size_t o_in = wl.add(in_bytes);
  size_t o_tq = wl.add(4 * (size_t)std::max<int64_t>(T, 1));
  size_t o_out = wl.add(4 * num_queries);
  void* ws = nullptr;
  st = ws_reserve(ctx, 0, wl.size, &ws);
  if (st) return st;
  char* wb = (char*)ws;
  char* din = wb + o_in;
  st = h2d_block(ctx, din, hp, in_bytes);
  if (st) return st;
  int32_t* dcounts = mem == GVOX_DEVICE ? counts : (int32_t*)(wb + o_out);
  CK(cudaMemsetAsync(dcounts, 0, 4 * num_queries, ctx->stream));
  if (T > 0) {
    launch_tile_map((const int32_t*)(din + o_ts), num_queries, (int32_t*)(wb + o_tq), ctx->stream);
    TimerScope ts(ctx, GVOX_TIMER_OVERLAP);
    launch_overlap_union((const CloudDev* const*)(din + o_cl), (const MapDev* const*)(din + o_mp),
                         (const UnionQueryDev*)(din + o_q), (const UnionMemberDev*)(din + o_m),
                         (const int32_t*)(din + o_ts), (const int32_t*)(wb + o_tq), T, tile_pts,
                         (const double*)(din + o_pose), level, dcounts, ctx->stream);
  }
  CK_LAUNCH(fn);
  if (mem == GVOX_HOST) {
    CK(cudaMemcpyAsync(counts, dcounts, 4 * num_queries, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return GVOX_OK;
}

gvox_status gvox_keyframe_update(const double* overlap, int32_t K, int32_t n_odom,
                                 double min_overlap, uint8_t* remove) {
  const char* fn = "gvox_keyframe_update";
  if (K < 1 || n_odom < 1) return fail(GVOX_ERR_INVALID, "%s: need K >= 1 and n_odom >= 1", fn);
  if (!overlap || !remove) return fail(GVOX_ERR_INVALID, "%s: NULL argument", fn);
  for (int64_t i = 0; i < (int64_t)K * K; ++i)
    if (!std::isfinite(overlap[i]))
      return fail(GVOX_ERR_INVALID, "%s: overlap[%lld] is not finite", fn, (long long)i);
  const int latest = K - 1;
  std::vector<uint8_t> rm(K, 0);
  // 1. keyframes overlapping the latest one by less than min_overlap
  for (int i = 0; i < latest; ++i)
    if (overlap[(int64_t)i * K + latest] < min_overlap) rm[i] = 1;
  // 2. one score-based removal while more than n_odom keyframes remain
  int remaining = 0;
  for (int i = 0; i < K; ++i) remaining += !rm[i];
  if (remaining > n_odom) {
    int best = -1;
    double best_s = 0.0;
    for (int i = 0; i < latest; ++i) {
      if (rm[i]) continue;
      double sum = 0.0;
      for (int j = 0; j < latest; ++j)
        if (j != i && !rm[j]) sum += 1.0 - overlap[(int64_t)i * K + j];
      const double s = overlap[(int64_t)i * K + latest] * sum;
      if (best < 0 || s < best_s) {
        best = i;
        best_s = s;
      }
    }
    if (best >= 0) rm[best] = 1;
  }
  std::memcpy(remove, rm.data(), K);
  return GVOX_OK;
}

gvox_status gvox_keyframe_insert_test(int64_t count, int64_t n, int32_t num, int32_t den,
                                      int32_t* insert) {
  const char* fn = "gvox_keyframe_insert_test";
  if (!insert) return fail(GVOX_ERR_INVALID, "%s: NULL argument", fn);
  if (count < 0 || n < 0 || count > n)
    return fail(GVOX_ERR_INVALID, "%s: need 0 <= count <= n (count %lld, n %lld)", fn,
                (long long)count, (long long)n);
  if (num < 0 || den <= 0) return fail(GVOX_ERR_INVALID, "%s: need num >= 0 and den > 0", fn);
  // insert when the union overlap count / n is SMALLER than num / den;
  // in integers (n <= 2^62 / den is far beyond any cloud)
  *insert = ((__int128)den * count < (__int128)num * n) ? 1 : 0;
  return GVOX_OK;
}

gvox_status gvox_keyframe_update_counts(const int64_t* counts, const int64_t* sizes, int32_t K,
                                        int32_t n_odom, double min_overlap, uint8_t* remove,
                                        double* overlap_out) {
  const char* fn = "gvox_keyframe_update_counts";
  if (K < 1) return fail(GVOX_ERR_INVALID, "%s: need K >= 1", fn);
  if (!counts || !sizes || !remove) return fail(GVOX_ERR_INVALID, "%s: NULL argument", fn);
  std::vector<double> o((size_t)K * K);
  for (int i = 0; i < K; ++i) {
    if (sizes[i] < 0) return fail(GVOX_ERR_INVALID, "%s: sizes[%d] < 0", fn, i);
    for (int j = 0; j < K; ++j) {
      const int64_t c = counts[(int64_t)i * K + j];
      if (c < 0 || c > sizes[i])
        return fail(GVOX_ERR_INVALID, "%s: counts[%d][%d] = %lld outside [0, sizes[%d]]", fn, i, j,
                    (long long)c, i);
      // P:280 overlap rate o(i, j): the fraction of keyframe i's points in j's voxels
      o[(size_t)i * K + j] = sizes[i] ? (double)c / (double)sizes[i] : 0.0;
    }
  }
  if (overlap_out) std::memcpy(overlap_out, o.data(), o.size() * sizeof(double));
  return gvox_keyframe_update(o.data(), K, n_odom, min_overlap, remove);
}

// ------------------------------------------------------------ registration
namespace {
constexpr int kRegMinTiles = 32;
}
gvox_status gvox_register_batch(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                int64_t num_clouds, const gvox_map* const* maps, int64_t num_maps,
                                const gvox_factor* factors, int64_t num_factors,
                                const double* poses, int64_t num_poses,
                                const gvox_register_params* params, double* poses_out,
                                gvox_register_result* results, double* error_history, int mem) {
  const char* fn = "gvox_register_batch";
  if (!ctx) return fail(GVOX_ERR_INVALID, "%s: ctx is NULL", fn);
  if (num_factors < 0 || num_poses < 0) return fail(GVOX_ERR_INVALID, "%s: negative size", fn);
  if (!params || !poses_out || !results || (num_factors > 0 && (!clouds || !maps || !factors || !poses)))
    return fail(GVOX_ERR_INVALID, "%s: NULL argument", fn);
  if (mem != GVOX_HOST && mem != GVOX_DEVICE)
    return fail(GVOX_ERR_INVALID, "%s: mem must be GVOX_HOST or GVOX_DEVICE", fn);
  const gvox_register_params P = *params;
  if (P.max_iterations < 1 || P.max_iterations > 1000)
    return fail(GVOX_ERR_INVALID, "%s: max_iterations %d outside [1, 1000]", fn, P.max_iterations);
  if (!(P.lambda >= 0.0) || !std::isfinite(P.lambda) || !(P.eps_rot >= 0.0) ||
      !(P.eps_trans >= 0.0) || std::isnan(P.eps_rot) || std::isnan(P.eps_trans))
    return fail(GVOX_ERR_INVALID, "%s: lambda, eps_rot, eps_trans must be >= 0 (lambda finite)", fn);
  gvox_status st = validate_factors(fn, clouds, num_clouds, maps, num_maps, factors, num_factors,
                                    poses, num_poses);
  if (st) return st;
  // ---- problems: one per variable pose (a factor's pose_i), ascending pose
  std::vector<int32_t> nf(num_poses, 0);
  for (int64_t f = 0; f < num_factors; ++f) {
    if (factors[f].flags & GVOX_F_ERROR_ONLY)
      return fail(GVOX_ERR_INVALID, "%s: factor %lld has GVOX_F_ERROR_ONLY (the solve needs H, b)",
                  fn, (long long)f);
    if (factors[f].pose_i == factors[f].pose_j)
      return fail(GVOX_ERR_INVALID, "%s: factor %lld has pose_i == pose_j", fn, (long long)f);
    ++nf[factors[f].pose_i];
  }
  for (int64_t f = 0; f < num_factors; ++f)
    if (nf[factors[f].pose_j])
      return fail(GVOX_ERR_INVALID,
                  "%s: factor %lld: pose_j %d is the variable pose of another factor (joint "
                  "multi-pose systems are not supported)", fn, (long long)f, factors[f].pose_j);
  std::vector<RegProblem> probs;
  std::vector<int32_t> pstart(num_poses + 1, 0);
  for (int64_t v = 0; v < num_poses; ++v) pstart[v + 1] = pstart[v] + nf[v];
  std::vector<int32_t> reg_f(std::max<int64_t>(num_factors, 1));
  {
    std::vector<int32_t> fill(pstart.begin(), pstart.end() - 1);
    for (int64_t f = 0; f < num_factors; ++f) reg_f[fill[factors[f].pose_i]++] = (int32_t)f;
  }
  for (int64_t v = 0; v < num_poses; ++v)
    if (nf[v]) probs.push_back(RegProblem{(int32_t)v, pstart[v], pstart[v + 1], 0});
  const int64_t NP = (int64_t)probs.size();
  DeviceGuard g(ctx->device);
  LinPlan plan;
  if (num_factors > 0) {
    // registration batches are small (one odometry step: ~10 factors): tiles
    // of >= 32 per factor keep every SM busy in the latency-bound loop
    st = plan_linearize(fn, clouds, maps, factors, num_factors,
                        std::getenv("GVOX_LIN_GENERIC") == nullptr, &plan,
                        std::getenv("GVOX_REG_MIN_TILES") ? std::max(1, std::atoi(std::getenv("GVOX_REG_MIN_TILES")))
                                                          : kRegMinTiles);
    if (st) return st;
  }
  const int64_t T = num_factors > 0 ? plan.tstart[num_factors] : 0;
  // ---- initial state
  std::vector<gvox_register_result> res0(std::max<int64_t>(num_poses, 1));
  std::memset(res0.data(), 0, sizeof(gvox_register_result) * res0.size());
  for (const RegProblem& q : probs) res0[q.pose].status = GVOX_REG_MAX_ITER;
  RegControl c0{};
  c0.iter = 0;
  c0.max_iter = P.max_iterations;
  c0.lambda = P.lambda;
  c0.eps_rot = P.eps_rot;
  c0.eps_trans = P.eps_trans;
  const int64_t HN = error_history ? (int64_t)P.max_iterations * num_poses : 0;
  // ---- one serialized input block; the OUTPUT regions (poses, results,
  // history) are contiguous at its start so a host D2H is one copy
  Layout lay;
  size_t o_pose = lay.add(96 * num_poses);
  size_t o_res = lay.add(sizeof(gvox_register_result) * num_poses);
  size_t o_hist = lay.add(8 * HN);
  const size_t out_bytes = lay.size;
  size_t o_ctrl = lay.add(sizeof(RegControl));
  size_t o_act = lay.add(4 * std::max<int64_t>(NP, 1));
  size_t o_prob = lay.add(sizeof(RegProblem) * std::max<int64_t>(NP, 1));
  size_t o_rf = lay.add(4 * reg_f.size());
  size_t o_fac = lay.add(sizeof(FactorDev) * num_factors);
  size_t o_ts = lay.add(4 * (num_factors + 1));
  size_t o_cl = lay.add(8 * num_clouds);
  size_t o_mp = lay.add(8 * num_maps);
  const size_t in_bytes = lay.size;
  void* pin = nullptr;
  st = pin_reserve(ctx, in_bytes, &pin);
  if (st) return st;
  char* hp = (char*)pin;
  std::memset(hp, 0, in_bytes);
  if (num_poses) std::memcpy(hp + o_pose, poses, 96 * num_poses);
  if (num_poses) std::memcpy(hp + o_res, res0.data(), sizeof(gvox_register_result) * num_poses);
  std::memcpy(hp + o_ctrl, &c0, sizeof(c0));
  for (int64_t k = 0; k < NP; ++k) ((int32_t*)(hp + o_act))[k] = 1;
  if (NP) std::memcpy(hp + o_prob, probs.data(), sizeof(RegProblem) * NP);
  std::memcpy(hp + o_rf, reg_f.data(), 4 * reg_f.size());
  if (num_factors) {
    std::memcpy(hp + o_fac, plan.fdev.data(), sizeof(FactorDev) * num_factors);
    std::memcpy(hp + o_ts, plan.tstart.data(), 4 * (num_factors + 1));
  }
  for (int64_t i = 0; i < num_clouds; ++i) ((const CloudDev**)(hp + o_cl))[i] = clouds[i] ? clouds[i]->dev : nullptr;
  for (int64_t i = 0; i < num_maps; ++i) ((const MapDev**)(hp + o_mp))[i] = maps[i] ? maps[i]->dev : nullptr;
  Layout wl;
  size_t o_in = wl.add(in_bytes);
  size_t o_part = wl.add(8 * kPartialStride * (size_t)std::max<int64_t>(T, 1));
  size_t o_tf = wl.add(4 * (size_t)std::max<int64_t>(T, 1));
  size_t o_acc = wl.add(sizeof(gvox_factor_accum) * std::max<int64_t>(num_factors, 1));
  void* ws = nullptr;
  st = ws_reserve(ctx, 0, wl.size, &ws);
  if (st) return st;
  char* wb = (char*)ws;
  char* din = wb + o_in;
  st = h2d_block(ctx, din, hp, in_bytes);
  if (st) return st;
  if (NP > 0) {
    launch_tile_map((const int32_t*)(din + o_ts), num_factors, (int32_t*)(wb + o_tf), ctx->stream);
    CK_LAUNCH("register tile map");
    auto body = [&](cudaStream_t sm, cudaGraphConditionalHandle cond) {
      launch_linearize((const CloudDev* const*)(din + o_cl), (const MapDev* const*)(din + o_mp),
                       (const FactorDev*)(din + o_fac), (const int32_t*)(din + o_ts), num_factors, T,
                       0, plan.max_levels, (const double*)(din + o_pose), (double*)(wb + o_part),
                       (int32_t*)(wb + o_tf), nullptr, plan.all_dense, plan.fast, plan.validate, sm);
      launch_reduce((const FactorDev*)(din + o_fac), (const int32_t*)(din + o_ts), num_factors,
                    (const double*)(din + o_pose), (const double*)(wb + o_part), nullptr,
                    (gvox_factor_accum*)(wb + o_acc), sm);
      launch_gn_step((const RegProblem*)(din + o_prob), (int32_t)NP, (const int32_t*)(din + o_rf),
                     (const FactorDev*)(din + o_fac), (const gvox_factor_accum*)(wb + o_acc),
                     (double*)(din + o_pose), (gvox_register_result*)(din + o_res),
                     (int32_t*)(din + o_act), (RegControl*)(din + o_ctrl),
                     HN ? (double*)(din + o_hist) : nullptr, num_poses, cond, sm);
    };
    if (std::getenv("GVOX_REG_EAGER")) {
      // profiling aid (ncu does not see kernels inside conditional graph
      // nodes): max_iterations plain launches; stopped problems are skipped
      // by the solve kernel, so results are identical
      TimerScope ts(ctx, GVOX_TIMER_REGISTER);
      for (int it = 0; it < P.max_iterations; ++it) body(ctx->stream, 0);
      CK_LAUNCH("register loop (eager)");
    } else {
    if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    // ---- the loop: a WHILE node whose body is linearize -> reduce -> solve
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    CK(cudaGraphCreate(&graph, 0));
    std::unique_ptr<CUgraph_st, void (*)(cudaGraph_t)> graph_guard(graph, [](cudaGraph_t gr) { cudaGraphDestroy(gr); });
    cudaGraphConditionalHandle cond;
    CK(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
    cudaGraph_t body_graph = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(ctx->cap_stream, body_graph, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    body(ctx->cap_stream, cond);
    cudaGraph_t captured = nullptr;
    cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &captured);
    if (ce != cudaSuccess) return cuda_fail(ce, "register loop capture");
    CK_LAUNCH("register loop capture");
    CK(cudaGraphInstantiate(&exec, graph, 0));
    {
      TimerScope ts(ctx, GVOX_TIMER_REGISTER);
      cudaError_t le = cudaGraphLaunch(exec, ctx->stream);
      if (le != cudaSuccess) {
        cudaGraphExecDestroy(exec);
        return cuda_fail(le, "register loop launch");
      }
    }
    note_launch();
    CK(cudaGraphExecDestroy(exec));  // freed asynchronously once the launch completes
    }
  }
  // ---- outputs
  if (mem == GVOX_DEVICE) {
    if (num_poses) {
      CK(cudaMemcpyAsync(poses_out, din + o_pose, 96 * num_poses, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(results, din + o_res, sizeof(gvox_register_result) * num_poses,
                         cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (HN) CK(cudaMemcpyAsync(error_history, din + o_hist, 8 * HN, cudaMemcpyDeviceToDevice, ctx->stream));
    return GVOX_OK;
  }
  if (ctx->pin_out_bytes < out_bytes) {
    if (ctx->pin_out) CK(cudaFreeHost(ctx->pin_out));
    ctx->pin_out = nullptr;
    size_t nb = align_up(std::max(out_bytes, ctx->pin_out_bytes * 3 / 2), 1 << 16);
    cudaError_t e = cudaHostAlloc(&ctx->pin_out, nb, cudaHostAllocDefault);
    if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc");
    ctx->pin_out_bytes = nb;
  }
  CK(cudaMemcpyAsync(ctx->pin_out, din, out_bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const char* ho = (const char*)ctx->pin_out;
  if (num_poses) {
    std::memcpy(poses_out, ho + o_pose, 96 * num_poses);
    std::memcpy(results, ho + o_res, sizeof(gvox_register_result) * num_poses);
  }
  if (HN) std::memcpy(error_history, ho + o_hist, 8 * HN);
  return GVOX_OK;
}

// ------------------------------------------------------------ global system
gvox_status gvox_solve_global(gvox_ctx* ctx, const gvox_factor* factors, int64_t num_factors,
                              const gvox_factor_accum* accum, const double* poses,
                              int64_t num_poses, const uint8_t* fixed,
                              const gvox_global_params* params, double* delta, double* H_dense,
                              double* b_dense, gvox_global_result* result, int mem) {
  const char* fn = "gvox_solve_global";
  if (!ctx) return fail(GVOX_ERR_INVALID, "%s: ctx is NULL", fn);
  if (num_factors < 0 || num_poses < 0) return fail(GVOX_ERR_INVALID, "%s: negative size", fn);
  if (!params || !fixed || !delta || !result || (num_poses > 0 && !poses) ||
      (num_factors > 0 && (!factors || !accum)))
    return fail(GVOX_ERR_INVALID, "%s: NULL argument", fn);
  if (mem != GVOX_HOST && mem != GVOX_DEVICE)
    return fail(GVOX_ERR_INVALID, "%s: mem must be GVOX_HOST or GVOX_DEVICE", fn);
  const gvox_global_params P = *params;
  if (P.max_iterations < 1 || !(P.tol >= 0.0) || !(P.lambda >= 0.0) || !std::isfinite(P.lambda))
    return fail(GVOX_ERR_INVALID, "%s: need max_iterations >= 1, tol >= 0, finite lambda >= 0", fn);
  gvox_status st = validate_factors(fn, nullptr, 0, nullptr, 0, factors, num_factors, poses, num_poses);
  if (st) return st;
  // ---- variables and the block pattern (host)
  std::vector<int32_t> var_of(num_poses, -1);
  int32_t V = 0;
  bool any_fixed = false;
  for (int64_t i = 0; i < num_poses; ++i) {
    if (fixed[i]) any_fixed = true;
    else var_of[i] = V++;
  }
  std::memset(result, 0, sizeof(*result));
  result->num_variables = V;
  if (V > 0 && !any_fixed && P.lambda == 0.0)
    return fail(GVOX_ERR_INVALID, "%s: no fixed pose and lambda = 0 (the gauge is free)", fn);
  struct Ent {
    int32_t row, col, code;
  };
  std::vector<Ent> ent;
  ent.reserve(4 * num_factors + V);
  for (int32_t v = 0; v < V; ++v) ent.push_back({v, v, -1});  // every variable has its diagonal block
  std::vector<std::vector<int32_t>> g(V);
  for (int64_t f = 0; f < num_factors; ++f) {
    const int32_t vi = var_of[factors[f].pose_i], vj = var_of[factors[f].pose_j];
    const int32_t c = (int32_t)(f << 2);
    if (vi >= 0) {
      ent.push_back({vi, vi, c | 0});
      g[vi].push_back((int32_t)(f << 1) | 0);
    }
    if (vi >= 0 && vj >= 0) {
      ent.push_back({vi, vj, c | 1});
      ent.push_back({vj, vi, c | 2});
    }
    if (vj >= 0) {
      ent.push_back({vj, vj, c | 3});
      g[vj].push_back((int32_t)(f << 1) | 1);
    }
  }
  if (num_factors > (1 << 28)) return fail(GVOX_ERR_INVALID, "%s: too many factors", fn);
  std::stable_sort(ent.begin(), ent.end(), [](const Ent& a, const Ent& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  std::vector<int32_t> row_start(V + 1, 0), col, cstart, contrib, diag_block(V, -1);
  std::vector<uint8_t> is_diag;
  for (size_t k = 0; k < ent.size();) {
    size_t e = k;
    const int32_t nb = (int32_t)col.size();
    col.push_back(ent[k].col);
    is_diag.push_back(ent[k].row == ent[k].col);
    if (ent[k].row == ent[k].col) diag_block[ent[k].row] = nb;
    cstart.push_back((int32_t)contrib.size());
    while (e < ent.size() && ent[e].row == ent[k].row && ent[e].col == ent[k].col) {
      if (ent[e].code >= 0) contrib.push_back(ent[e].code);
      ++e;
    }
    row_start[ent[k].row + 1] = nb + 1;
    k = e;
  }
  for (int32_t v = 0; v < V; ++v) row_start[v + 1] = std::max(row_start[v + 1], row_start[v]);
  const int64_t NB = (int64_t)col.size();
  cstart.push_back((int32_t)contrib.size());
  std::vector<int32_t> gstart(V + 1, 0), glist;
  for (int32_t v = 0; v < V; ++v) {
    glist.insert(glist.end(), g[v].begin(), g[v].end());
    gstart[v + 1] = (int32_t)glist.size();
  }
  result->num_blocks = (int32_t)NB;
  // SpMV work units of the persistent PCG: each block row cut into chunks of at
  // most kPcgChunk blocks (GVOX_PCG_CHUNK; 0 = one chunk per row), so no warp
  // walks a whole long row while the others wait at the barrier
  int pcg_chunk = 64;
  if (const char* e = std::getenv("GVOX_PCG_CHUNK")) pcg_chunk = std::atoi(e);
  std::vector<int32_t> chunk_row, chunk_b0, row_chunk(V + 1, 0);
  for (int32_t v = 0; v < V; ++v) {
    row_chunk[v] = (int32_t)chunk_row.size();
    const int32_t b0 = row_start[v], b1 = row_start[v + 1];
    const int32_t step = pcg_chunk > 0 ? pcg_chunk : std::max(b1 - b0, 1);
    for (int32_t b = b0; b < b1 || b == b0; b += step) {  // (an empty row still gets one chunk)
      chunk_row.push_back(v);
      chunk_b0.push_back(b);
      if (b1 <= b0) break;
    }
  }
  row_chunk[V] = (int32_t)chunk_row.size();
  const int64_t NC = (int64_t)chunk_row.size();
  DeviceGuard dg(ctx->device);
  // ---- one input block
  std::vector<FactorDev> fdev(num_factors);
  for (int64_t f = 0; f < num_factors; ++f)
    fdev[f] = FactorDev{factors[f].source_cloud, factors[f].target_map, factors[f].pose_i,
                        factors[f].pose_j, factors[f].flags, 0, 0};
  Layout lay;
  size_t o_pose = lay.add(96 * num_poses);
  size_t o_fac = lay.add(sizeof(FactorDev) * num_factors);
  size_t o_rs = lay.add(4 * row_start.size());
  size_t o_col = lay.add(4 * col.size());
  size_t o_cs = lay.add(4 * cstart.size());
  size_t o_ct = lay.add(4 * std::max<size_t>(contrib.size(), 1));
  size_t o_gs = lay.add(4 * gstart.size());
  size_t o_gl = lay.add(4 * std::max<size_t>(glist.size(), 1));
  size_t o_dg = lay.add(4 * std::max<int32_t>(V, 1));
  size_t o_isd = lay.add(std::max<size_t>(is_diag.size(), 1));
  size_t o_vo = lay.add(4 * std::max<int64_t>(num_poses, 1));
  size_t o_acc = lay.add(mem == GVOX_HOST ? sizeof(gvox_factor_accum) * num_factors : 0);
  size_t o_crow = lay.add(4 * std::max<int64_t>(NC, 1));
  size_t o_cb0 = lay.add(4 * std::max<int64_t>(NC, 1));
  size_t o_rch = lay.add(4 * row_chunk.size());
  const size_t in_bytes = lay.size;
  void* pin = nullptr;
  st = pin_reserve(ctx, in_bytes, &pin);
  if (st) return st;
  char* hp = (char*)pin;
  if (num_poses) std::memcpy(hp + o_pose, poses, 96 * num_poses);
  if (num_factors) std::memcpy(hp + o_fac, fdev.data(), sizeof(FactorDev) * num_factors);
  std::memcpy(hp + o_rs, row_start.data(), 4 * row_start.size());
  if (!col.empty()) std::memcpy(hp + o_col, col.data(), 4 * col.size());
  std::memcpy(hp + o_cs, cstart.data(), 4 * cstart.size());
  if (!contrib.empty()) std::memcpy(hp + o_ct, contrib.data(), 4 * contrib.size());
  std::memcpy(hp + o_gs, gstart.data(), 4 * gstart.size());
  if (!glist.empty()) std::memcpy(hp + o_gl, glist.data(), 4 * glist.size());
  if (V) std::memcpy(hp + o_dg, diag_block.data(), 4 * V);
  if (!is_diag.empty()) std::memcpy(hp + o_isd, is_diag.data(), is_diag.size());
  if (num_poses) std::memcpy(hp + o_vo, var_of.data(), 4 * num_poses);
  if (mem == GVOX_HOST && num_factors) std::memcpy(hp + o_acc, accum, sizeof(gvox_factor_accum) * num_factors);
  if (NC) {
    std::memcpy(hp + o_crow, chunk_row.data(), 4 * NC);
    std::memcpy(hp + o_cb0, chunk_b0.data(), 4 * NC);
  }
  std::memcpy(hp + o_rch, row_chunk.data(), 4 * row_chunk.size());
  Layout wl;
  size_t o_in = wl.add(in_bytes);
  size_t o_rec = wl.add(sizeof(gvox_linear_factor) * std::max<int64_t>(num_factors, 1));
  size_t o_blk = wl.add(8 * 36 * std::max<int64_t>(NB, 1));
  const int64_t n6 = 6 * (int64_t)std::max<int32_t>(V, 1);
  size_t o_rhs = wl.add(8 * n6), o_x = wl.add(8 * n6), o_r = wl.add(8 * n6), o_z = wl.add(8 * n6);
  size_t o_p = wl.add(8 * n6), o_q = wl.add(8 * n6), o_pq = wl.add(8 * (n6 / 6));
  size_t o_pb = wl.add(8 * (n6 / 6));
  size_t o_minv = wl.add(8 * 36 * (n6 / 6));
  size_t o_st = wl.add(sizeof(PcgState) + 16);
  size_t o_qpart = wl.add(8 * 6 * std::max<int64_t>(NC, 1));
  size_t o_pc = wl.add(8 * std::max<int64_t>(NC, 1));
  size_t o_dl = wl.add(mem == GVOX_HOST ? 48 * (size_t)std::max<int64_t>(num_poses, 1) : 0);
  void* ws = nullptr;
  st = ws_reserve(ctx, 0, wl.size, &ws);
  if (st) return st;
  char* wb = (char*)ws;
  char* din = wb + o_in;
  st = h2d_block(ctx, din, hp, in_bytes);
  if (st) return st;
  int32_t* dbad = (int32_t*)(wb + o_st + sizeof(PcgState));
  PcgState* dst = (PcgState*)(wb + o_st);
  CK(cudaMemsetAsync(wb + o_st, 0, sizeof(PcgState) + 16, ctx->stream));
  const gvox_factor_accum* dacc = mem == GVOX_HOST ? (const gvox_factor_accum*)(din + o_acc) : accum;
  double* ddelta = mem == GVOX_DEVICE ? delta : (double*)(wb + o_dl);
  {
    TimerScope ts(ctx, GVOX_TIMER_SOLVE);
    launch_expand((const FactorDev*)(din + o_fac), num_factors, (const double*)(din + o_pose), dacc,
                  (gvox_linear_factor*)(wb + o_rec), ctx->stream);
    launch_assemble((const gvox_linear_factor*)(wb + o_rec), (const int32_t*)(din + o_cs),
                    (const int32_t*)(din + o_ct), NB, (const uint8_t*)(din + o_isd), P.lambda,
                    (double*)(wb + o_blk), (const int32_t*)(din + o_gs), (const int32_t*)(din + o_gl),
                    V, (double*)(wb + o_rhs), (const int32_t*)(din + o_dg), (double*)(wb + o_minv),
                    dbad, ctx->stream);
    CK_LAUNCH("global assemble");
    if (V > 0 && std::getenv("GVOX_PCG_GRAPH") == nullptr &&
        launch_pcg_cluster((const double*)(wb + o_blk), (const int32_t*)(din + o_rs),
                           (const int32_t*)(din + o_col), V, NB, (const double*)(wb + o_minv),
                           (const double*)(wb + o_rhs), (double*)(wb + o_x), (double*)(wb + o_r),
                           (double*)(wb + o_z), (double*)(wb + o_p), (double*)(wb + o_q), dst,
                           P.max_iterations, P.tol, ctx->stream)) {
      // (the whole PCG on one thread-block cluster: hardware cluster barriers)
      CK_LAUNCH("PCG (cluster)");
    } else if (V > 0 && std::getenv("GVOX_PCG_GRAPH") == nullptr) {
      // one cooperative persistent kernel runs the whole PCG (grid barriers)
      launch_pcg_persistent((const double*)(wb + o_blk), (const int32_t*)(din + o_rs),
                            (const int32_t*)(din + o_col), V, (const double*)(wb + o_minv),
                            (const double*)(wb + o_rhs), (double*)(wb + o_x), (double*)(wb + o_r),
                            (double*)(wb + o_z), (double*)(wb + o_p), (double*)(wb + o_q),
                            (double*)(wb + o_pq), (double*)(wb + o_pb), dst, P.max_iterations,
                            P.tol, (const int32_t*)(din + o_crow), (const int32_t*)(din + o_cb0),
                            (const int32_t*)(din + o_rch), NC, (double*)(wb + o_qpart),
                            (double*)(wb + o_pc), ctx->stream);
      CK_LAUNCH("PCG (persistent)");
    } else if (V > 0) {
      launch_pcg_init((const double*)(wb + o_rhs), (const double*)(wb + o_minv), V, (double*)(wb + o_x),
                      (double*)(wb + o_r), (double*)(wb + o_z), (double*)(wb + o_p), dst, ctx->stream);
      if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
      cudaGraph_t graph = nullptr;
      cudaGraphExec_t exec = nullptr;
      CK(cudaGraphCreate(&graph, 0));
      std::unique_ptr<CUgraph_st, void (*)(cudaGraph_t)> guard(graph, [](cudaGraph_t gr) { cudaGraphDestroy(gr); });
      cudaGraphConditionalHandle cond;
      CK(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = cond;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t node;
      CK(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
      CK(cudaStreamBeginCaptureToGraph(ctx->cap_stream, cp.conditional.phGraph_out[0], nullptr, nullptr,
                                       0, cudaStreamCaptureModeThreadLocal));
      launch_pcg_iteration((const double*)(wb + o_blk), (const int32_t*)(din + o_rs),
                           (const int32_t*)(din + o_col), V, (const double*)(wb + o_minv),
                           (double*)(wb + o_x), (double*)(wb + o_r), (double*)(wb + o_z),
                           (double*)(wb + o_p), (double*)(wb + o_q), (double*)(wb + o_pq), dst,
                           P.max_iterations, P.tol, cond, ctx->cap_stream);
      cudaGraph_t captured = nullptr;
      cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &captured);
      if (ce != cudaSuccess) return cuda_fail(ce, "PCG loop capture");
      CK(cudaGraphInstantiate(&exec, graph, 0));
      cudaError_t le = cudaGraphLaunch(exec, ctx->stream);
      cudaGraphExecDestroy(exec);
      if (le != cudaSuccess) return cuda_fail(le, "PCG loop launch");
      note_launch();
    }
    if (num_poses > 0) {
      if (V > 0) {
        launch_scatter_delta((const double*)(wb + o_x), (const int32_t*)(din + o_vo), num_poses,
                             ddelta, ctx->stream);
      } else {
        CK(cudaMemsetAsync(ddelta, 0, 48 * num_poses, ctx->stream));
      }
    }
  }
  CK_LAUNCH(fn);
  // ---- results (always synchronizes: the result struct is host memory)
  PcgState hs{};
  int32_t hbad = 0;
  CK(cudaMemcpyAsync(&hs, dst, sizeof(PcgState), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&hbad, dbad, 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (mem == GVOX_HOST && num_poses)
    CK(cudaMemcpyAsync(delta, ddelta, 48 * num_poses, cudaMemcpyDeviceToHost, ctx->stream));
  std::vector<double> hblk, hrhs;
  if (H_dense && V > 0) {
    hblk.resize(36 * NB);
    CK(cudaMemcpyAsync(hblk.data(), wb + o_blk, 8 * 36 * NB, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (b_dense && V > 0) {
    hrhs.resize(6 * V);
    CK(cudaMemcpyAsync(hrhs.data(), wb + o_rhs, 8 * 6 * V, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (hbad) return fail(GVOX_ERR_INVALID, "%s: a diagonal block is not positive definite", fn);
  result->iterations = hs.iter;
  result->residual_initial = hs.r0;
  result->residual_final = hs.res;
  result->converged = V == 0 || hs.res <= P.tol * hs.r0;
  if (H_dense && V > 0) {
    const int64_t D = 6 * (int64_t)V;
    std::memset(H_dense, 0, 8 * D * D);
    for (int32_t v = 0; v < V; ++v)
      for (int32_t b = row_start[v]; b < row_start[v + 1]; ++b)
        for (int e = 0; e < 36; ++e)
          H_dense[(6 * (int64_t)v + e / 6) * D + 6 * (int64_t)col[b] + e % 6] = hblk[36 * b + e];
  }
  if (b_dense && V > 0)
    for (int64_t t = 0; t < 6 * (int64_t)V; ++t) b_dense[t] = -hrhs[t];
  return GVOX_OK;
}

gvox_status gvox_optimize_global(gvox_ctx* ctx, const gvox_cloud* const* clouds,
                                 int64_t num_clouds, const gvox_map* const* maps, int64_t num_maps,
                                 const gvox_factor* factors, int64_t num_factors,
                                 const double* poses, int64_t num_poses, const uint8_t* fixed,
                                 const gvox_optimize_params* params, double* poses_out,
                                 double* error_history, gvox_optimize_result* result, int mem) {
  const char* fn = "gvox_optimize_global";
  if (!ctx) return fail(GVOX_ERR_INVALID, "%s: ctx is NULL", fn);
  if (!params || !result || !poses_out || !fixed || (num_poses > 0 && !poses))
    return fail(GVOX_ERR_INVALID, "%s: NULL argument", fn);
  if (num_poses < 0 || num_factors < 0) return fail(GVOX_ERR_INVALID, "%s: negative size", fn);
  if (mem != GVOX_HOST && mem != GVOX_DEVICE)
    return fail(GVOX_ERR_INVALID, "%s: mem must be GVOX_HOST or GVOX_DEVICE", fn);
  const gvox_optimize_params P = *params;
  if (P.max_iterations < 1 || P.max_iterations > 1000 || P.pcg_max_iterations < 1 ||
      !(P.eps_rot >= 0.0) || !(P.eps_trans >= 0.0))
    return fail(GVOX_ERR_INVALID, "%s: bad iteration counts or tolerances", fn);
  std::memset(result, 0, sizeof(*result));
  DeviceGuard g(ctx->device);
  // device state: records, step, poses, two scalars (error, max |w|, max |rho|);
  // a dedicated allocation (the linearize / solve calls reuse the workspaces)
  const size_t acc_b = sizeof(gvox_factor_accum) * (size_t)std::max<int64_t>(num_factors, 1);
  const size_t pose_b = 96 * (size_t)std::max<int64_t>(num_poses, 1);
  std::shared_ptr<DevBuf> buf;
  gvox_status st = devbuf_alloc(acc_b + pose_b + 48 * (size_t)std::max<int64_t>(num_poses, 1) + 64,
                                ctx->device, ctx->stream, &buf);
  if (st) return st;
  char* b0 = (char*)buf->ptr;
  gvox_factor_accum* dacc = (gvox_factor_accum*)b0;
  double* dposes = (double*)(b0 + acc_b);
  double* ddelta = (double*)(b0 + acc_b + pose_b);
  double* dscal = (double*)(b0 + acc_b + pose_b + 48 * (size_t)std::max<int64_t>(num_poses, 1));
  std::vector<double> ph(poses, poses + 12 * num_poses);
  gvox_global_params gp{P.pcg_max_iterations, 0, P.pcg_tol, P.lambda};
  for (int it = 0; it < P.max_iterations; ++it) {
    st = linearize_impl(ctx, clouds, num_clouds, maps, num_maps, factors, num_factors, ph.data(),
                        num_poses, nullptr, dacc, GVOX_DEVICE, nullptr);
    if (st) return st;
    launch_sum_error(dacc, num_factors, dscal, ctx->stream);
    gvox_global_result gr;
    st = gvox_solve_global(ctx, factors, num_factors, dacc, ph.data(), num_poses, fixed, &gp, ddelta,
                           nullptr, nullptr, &gr, GVOX_DEVICE);
    if (st) return st;
    if (num_poses) {
      CK(cudaMemcpyAsync(dposes, ph.data(), 96 * num_poses, cudaMemcpyHostToDevice, ctx->stream));
      launch_apply_delta(dposes, ddelta, num_poses, dscal + 1, ctx->stream);
      CK(cudaMemcpyAsync(ph.data(), dposes, 96 * num_poses, cudaMemcpyDeviceToHost, ctx->stream));
    }
    double sc[3] = {0, 0, 0};
    CK(cudaMemcpyAsync(sc, dscal, num_poses ? 24 : 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK_LAUNCH(fn);
    if (it == 0) result->error_initial = sc[0];
    result->error_final = sc[0];
    if (error_history) error_history[it] = sc[0];
    result->iterations = it + 1;
    result->pcg_iterations += gr.iterations;
    result->last_step_rot = sc[1];
    result->last_step_trans = sc[2];
    if (sc[1] <= P.eps_rot && sc[2] <= P.eps_trans) {
      result->converged = 1;
      break;
    }
  }
  if (num_poses) {
    if (mem == GVOX_HOST) std::memcpy(poses_out, ph.data(), 96 * num_poses);
    else CK(cudaMemcpyAsync(poses_out, dposes, 96 * num_poses, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return GVOX_OK;
}

// ------------------------------------------------------------------ utilities
const char* gvox_status_string(gvox_status s) {
  switch (s) {
    case GVOX_OK: return "GVOX_OK";
    case GVOX_ERR_INVALID: return "GVOX_ERR_INVALID";
    case GVOX_ERR_RANGE: return "GVOX_ERR_RANGE";
    case GVOX_ERR_CUDA: return "GVOX_ERR_CUDA";
    case GVOX_ERR_NOMEM: return "GVOX_ERR_NOMEM";
  }
  return "GVOX_ERR_UNKNOWN";
}

const char* gvox_last_error(void) { return g_last_error.c_str(); }

int64_t gvox_launch_count(int reset) {
  int64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

int32_t gvox_last_linearize_variant(void) { return g_lin_variant; }

const char* gvox_version(void) { return "gvox 0.1 (sm_100a)"; }

}  // extern "C"
