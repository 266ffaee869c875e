// gen.cpp -- seeded synthetic LiDAR-shaped inputs for the VGICP hot path.
//
// Shared by the oracle side (tests) and the CUDA side (tests, bench).  It holds
// NONE of the method's arithmetic (no voxel keys, no relative poses, no
// residuals): it ray-casts a procedural world, downsamples, subsamples and
// emits Gaussian points (mean, GICP plane covariance, oriented normal).
// The recipe is SURVEY.md Sec.8(d) "Synthetic inputs", restated in DESIGN.md.
//
// Randomness is a counter-based SplitMix64 hash of (seed, stream, counter), so
// every value is independent of thread count and evaluation order.
//
// World: ground plane z = 0 plus one yaw-rotated box per 40 m block (15 % of
// blocks empty), footprint 6-18 m, height 3-20 m, random sub-metre offsets.
// Sensor: OS0-128-like: `rings` rings over -45..+45 deg elevation,
// `azimuths` steps, max range 60 m, Gaussian range noise sigma (1 cm default).
// Per point: normal = hit surface normal (jittered by ~0.02 rad to mimic k-NN
// estimation noise), oriented toward the capture viewpoint; covariance
// C = U diag(1e-3, 1, 1) U^T with U = [n, t1, t2] (GICP plane model).

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

inline uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline uint64_t rng(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return splitmix(seed ^ splitmix(stream ^ splitmix(ctr)));
}
inline double uni(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return (double)(rng(seed, stream, ctr) >> 11) * (1.0 / 9007199254740992.0);
}
inline double gauss(uint64_t seed, uint64_t stream, uint64_t ctr) {
  double u1 = uni(seed, stream, 2 * ctr), u2 = uni(seed, stream, 2 * ctr + 1);
  if (u1 < 1e-300) u1 = 1e-300;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

const double kBlock = 40.0;

struct Box {
  double cx, cy, hx, hy, h, c, s;  // centre, half extents, height, cos/sin yaw
  bool present;
};

struct World {
  uint64_t seed;
  int half_blocks;  // blocks span [-half_blocks, half_blocks) per axis
  std::vector<Box> boxes;
  const Box& at(int i, int j) const {
    return boxes[(size_t)(i + half_blocks) * (2 * half_blocks) + (j + half_blocks)];
  }
};

void make_world(World* w, uint64_t seed, int half_blocks) {
  w->seed = seed;
  w->half_blocks = half_blocks;
  int nb = 2 * half_blocks;
  w->boxes.resize((size_t)nb * nb);
  for (int i = -half_blocks; i < half_blocks; ++i)
    for (int j = -half_blocks; j < half_blocks; ++j) {
      uint64_t stream = (uint64_t)((i + half_blocks) * nb + (j + half_blocks)) + 1000;
      Box b;
      b.present = uni(seed, stream, 0) >= 0.15;
      double yaw = uni(seed, stream, 1) * 1.5707963267948966;
      b.c = std::cos(yaw);
      b.s = std::sin(yaw);
      b.hx = 0.5 * (6.0 + 12.0 * uni(seed, stream, 2));
      b.hy = 0.5 * (6.0 + 12.0 * uni(seed, stream, 3));
      b.h = 3.0 + 17.0 * uni(seed, stream, 4);
      b.cx = (i + 0.5) * kBlock + (uni(seed, stream, 5) - 0.5) * 6.0 + 0.37;
      b.cy = (j + 0.5) * kBlock + (uni(seed, stream, 6) - 0.5) * 6.0 + 0.61;
      w->boxes[(size_t)(i + half_blocks) * nb + (j + half_blocks)] = b;
    }
}

// Ray vs one box: returns entry distance (or +inf) and world normal.
double hit_box(const Box& b, const double o[3], const double d[3], double n_out[3]) {
  // into box frame (rotate by -yaw about z)
  double ox = o[0] - b.cx, oy = o[1] - b.cy;
  double lo[3] = {b.c * ox + b.s * oy, -b.s * ox + b.c * oy, o[2]};
  double ld[3] = {b.c * d[0] + b.s * d[1], -b.s * d[0] + b.c * d[1], d[2]};
  double mn[3] = {-b.hx, -b.hy, 0.0}, mx[3] = {b.hx, b.hy, b.h};
  double t0 = -1e300, t1 = 1e300;
  int axis = -1;
  double sign = 0;
  for (int a = 0; a < 3; ++a) {
    if (std::fabs(ld[a]) < 1e-15) {
      if (lo[a] < mn[a] || lo[a] > mx[a]) return INFINITY;
      continue;
    }
    double ta = (mn[a] - lo[a]) / ld[a], tb = (mx[a] - lo[a]) / ld[a];
    double sa = -1.0;
    if (ta > tb) {
      std::swap(ta, tb);
      sa = 1.0;
    }
    if (ta > t0) {
      t0 = ta;
      axis = a;
      sign = sa;
    }
    if (tb < t1) t1 = tb;
    if (t0 > t1) return INFINITY;
  }
  if (t0 <= 1e-9 || axis < 0) return INFINITY;  // origin inside or behind
  double ln[3] = {0, 0, 0};
  ln[axis] = sign;
  n_out[0] = b.c * ln[0] - b.s * ln[1];
  n_out[1] = b.s * ln[0] + b.c * ln[1];
  n_out[2] = ln[2];
  return t0;
}

struct Hit {
  double t;
  double n[3];
};

// Nearest hit among the ground plane and the boxes met along the ray: a 2D DDA
// over the 40 m block grid, stopping once a hit lies before the next cell.
Hit cast(const World& w, const double o[3], const double d[3], double max_range) {
  Hit h;
  h.t = INFINITY;
  if (d[2] < -1e-12) {
    double t = -o[2] / d[2];
    if (t > 0) {
      h.t = t;
      h.n[0] = 0;
      h.n[1] = 0;
      h.n[2] = 1;
    }
  }
  double tmax_ray = std::min(h.t, max_range);
  int hb = w.half_blocks;
  int ci = (int)std::floor(o[0] / kBlock), cj = (int)std::floor(o[1] / kBlock);
  int si = d[0] > 0 ? 1 : -1, sj = d[1] > 0 ? 1 : -1;
  double tdx = std::fabs(d[0]) > 1e-15 ? kBlock / std::fabs(d[0]) : INFINITY;
  double tdy = std::fabs(d[1]) > 1e-15 ? kBlock / std::fabs(d[1]) : INFINITY;
  double nx = (si > 0 ? (ci + 1) * kBlock - o[0] : o[0] - ci * kBlock);
  double ny = (sj > 0 ? (cj + 1) * kBlock - o[1] : o[1] - cj * kBlock);
  double tx = std::fabs(d[0]) > 1e-15 ? nx / std::fabs(d[0]) : INFINITY;
  double ty = std::fabs(d[1]) > 1e-15 ? ny / std::fabs(d[1]) : INFINITY;
  double tcell = 0.0;
  // boxes overhang their block by < 0: footprint stays inside the block, so a
  // ray only meets a box while inside that box's block.
  for (int step = 0; step < 64; ++step) {
    if (tcell > tmax_ray || tcell > h.t) break;
    if (ci >= -hb && ci < hb && cj >= -hb && cj < hb) {
      const Box& b = w.at(ci, cj);
      if (b.present) {
        double n[3];
        double t = hit_box(b, o, d, n);
        if (t < h.t) {
          h.t = t;
          h.n[0] = n[0];
          h.n[1] = n[1];
          h.n[2] = n[2];
        }
      }
    }
    if (tx < ty) {
      tcell = tx;
      tx += tdx;
      ci += si;
    } else {
      tcell = ty;
      ty += tdy;
      cj += sj;
    }
  }
  if (h.t > max_range) h.t = INFINITY;
  return h;
}

struct RawPoint {
  double p[3];  // in the output (cloud) frame
  double n[3];  // exact surface normal in the output frame, toward the viewpoint
  uint64_t id;  // (frame, ray) counter for the per-point jitter stream
};

// Row-major 3x4 pose helpers (generator-local; world <- sensor).
void pose_apply(const double* T, const double x[3], double y[3]) {
  for (int a = 0; a < 3; ++a) y[a] = T[a * 4] * x[0] + T[a * 4 + 1] * x[1] + T[a * 4 + 2] * x[2] + T[a * 4 + 3];
}
void rot_apply(const double* T, const double x[3], double y[3]) {
  for (int a = 0; a < 3; ++a) y[a] = T[a * 4] * x[0] + T[a * 4 + 1] * x[1] + T[a * 4 + 2] * x[2];
}
void rot_apply_t(const double* T, const double x[3], double y[3]) {
  for (int a = 0; a < 3; ++a) y[a] = T[a] * x[0] + T[4 + a] * x[1] + T[8 + a] * x[2];
}

// One scan from world pose Ts (world <- sensor); points expressed in the frame
// of world pose To (world <- output frame).
void scan(const World& w, const double* Ts, const double* To, int rings, int azimuths,
          double max_range, double sigma, uint64_t seed, uint64_t frame_id,
          std::vector<RawPoint>* out) {
  double o[3] = {Ts[3], Ts[7], Ts[11]};
  for (int r = 0; r < rings; ++r) {
    double el = (-45.0 + 90.0 * (rings > 1 ? (double)r / (rings - 1) : 0.5)) * M_PI / 180.0;
    for (int a = 0; a < azimuths; ++a) {
      double az = 2.0 * M_PI * ((double)a + 0.5) / azimuths;
      double ds[3] = {std::cos(el) * std::cos(az), std::cos(el) * std::sin(az), std::sin(el)};
      double dw[3];
      rot_apply(Ts, ds, dw);
      Hit h = cast(w, o, dw, max_range);
      if (!std::isfinite(h.t) || h.t < 0.5) continue;
      uint64_t ray = (uint64_t)r * azimuths + a;
      double t = h.t + sigma * gauss(seed, 7 + 131 * frame_id, ray);
      double pw[3] = {o[0] + t * dw[0], o[1] + t * dw[1], o[2] + t * dw[2]};
      RawPoint rp;
      double rel[3] = {pw[0] - To[3], pw[1] - To[7], pw[2] - To[11]};
      rot_apply_t(To, rel, rp.p);
      rot_apply_t(To, h.n, rp.n);  // exact surface normal; faces the sensor (front face)
      rp.id = frame_id * 0x100000000ull + ray;
      out->push_back(rp);
    }
  }
}

uint64_t spread3(uint64_t v) {  // 21 bits -> every third bit
  v &= 0x1FFFFF;
  v = (v | v << 32) & 0x1F00000000FFFFull;
  v = (v | v << 16) & 0x1F0000FF0000FFull;
  v = (v | v << 8) & 0x100F00F00F00F00Full;
  v = (v | v << 4) & 0x10C30C30C30C30C3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}

// Downsample (first point per ds_res cell), seeded subsample to exactly
// n_target (or all if fewer), order by Morton code of the 0.25 m cell
// (spatially coherent order, what a sorted voxel-grid downsampler emits), emit.
int64_t finish_cloud(std::vector<RawPoint>& raw, double ds_res, int64_t n_target, uint64_t seed,
                     uint64_t cloud_id, int order_random, float* mu, float* cov, float* nrm) {
  std::unordered_map<uint64_t, size_t> cell;
  cell.reserve(raw.size() * 2);
  std::vector<size_t> keep;
  const int64_t off = int64_t(1) << 20;
  for (size_t i = 0; i < raw.size(); ++i) {
    int64_t k[3];
    for (int c = 0; c < 3; ++c) k[c] = (int64_t)std::floor(raw[i].p[c] / ds_res) + off;
    uint64_t key = ((uint64_t)k[0] << 42) | ((uint64_t)k[1] << 21) | (uint64_t)k[2];
    if (cell.emplace(key, i).second) keep.push_back(i);
  }
  // seeded subsample: keep the n_target smallest random priorities
  std::vector<std::pair<uint64_t, size_t>> pri(keep.size());
  for (size_t i = 0; i < keep.size(); ++i) pri[i] = {rng(seed, 0x5EED0000ull + cloud_id, keep[i]), keep[i]};
  int64_t n = std::min<int64_t>(n_target, (int64_t)pri.size());
  if ((int64_t)pri.size() > n) {
    std::nth_element(pri.begin(), pri.begin() + n, pri.end());
    pri.resize(n);
  }
  std::vector<std::pair<uint64_t, size_t>> ord(n);
  for (int64_t i = 0; i < n; ++i) {
    const RawPoint& p = raw[pri[i].second];
    uint64_t code;
    if (order_random) {
      code = pri[i].first;
    } else {
      uint64_t k[3];
      for (int c = 0; c < 3; ++c) k[c] = (uint64_t)((int64_t)std::floor(p.p[c] / 0.25) + off);
      code = (spread3(k[0]) << 2) | (spread3(k[1]) << 1) | spread3(k[2]);
    }
    ord[i] = {code, pri[i].second};
  }
  std::sort(ord.begin(), ord.end());
  for (int64_t i = 0; i < n; ++i) {
    const RawPoint& p = raw[ord[i].second];
    // normal jitter (k-NN estimation noise, ~0.02 rad), kept on the viewpoint side
    double nv[3];
    for (int c = 0; c < 3; ++c) nv[c] = p.n[c] + 0.02 * gauss(seed, 9, 3 * p.id + c);
    double nn = std::sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
    double side = nv[0] * p.n[0] + nv[1] * p.n[1] + nv[2] * p.n[2];
    for (int c = 0; c < 3; ++c) nv[c] = (side < 0 ? -nv[c] : nv[c]) / nn;
    // C = U diag(1e-3, 1, 1) U^T = I - (1 - 1e-3) n n^T
    double e = 1.0 - 1e-3;
    double C[6] = {1 - e * nv[0] * nv[0], -e * nv[0] * nv[1], -e * nv[0] * nv[2],
                   1 - e * nv[1] * nv[1], -e * nv[1] * nv[2], 1 - e * nv[2] * nv[2]};
    for (int c = 0; c < 3; ++c) {
      mu[3 * i + c] = (float)p.p[c];
      nrm[3 * i + c] = (float)nv[c];
    }
    for (int c = 0; c < 6; ++c) cov[6 * i + c] = (float)C[c];
  }
  return n;
}

}  // namespace

extern "C" {

void* synth_world_create(uint64_t seed, int half_blocks) {
  World* w = new World;
  make_world(w, seed, half_blocks);
  return w;
}

void synth_world_free(void* w) { delete (World*)w; }

// Is (x, y) inside a box footprint (used by tests to keep paths on streets).
int synth_world_occupied(void* wp, double x, double y) {
  const World& w = *(World*)wp;
  int i = (int)std::floor(x / kBlock), j = (int)std::floor(y / kBlock);
  if (i < -w.half_blocks || i >= w.half_blocks || j < -w.half_blocks || j >= w.half_blocks) return 0;
  const Box& b = w.at(i, j);
  if (!b.present) return 0;
  double ox = x - b.cx, oy = y - b.cy;
  double lx = b.c * ox + b.s * oy, ly = -b.s * ox + b.c * oy;
  return std::fabs(lx) <= b.hx && std::fabs(ly) <= b.hy;
}

// Build `num_clouds` clouds.  Cloud c merges frames_per_cloud scans taken at
// world poses frame_poses[(c*fpc + f)*12] (world <- sensor), expressed in the
// frame of origin_poses[c*12]; downsampled at ds_res, subsampled to exactly
// n_target points (fewer if the scans have fewer cells).  Outputs are strided
// by n_target: mu[c*n_target*3], cov[c*n_target*6], nrm[c*n_target*3];
// counts[c] = points emitted.
void synth_make_clouds(void* wp, int64_t num_clouds, int frames_per_cloud,
                       const double* frame_poses, const double* origin_poses, int rings,
                       int azimuths, double max_range, double sigma, double ds_res,
                       int64_t n_target, uint64_t seed, uint64_t first_cloud_id, int order_random,
                       int num_threads, float* mu, float* cov, float* nrm, int64_t* counts) {
  const World& w = *(World*)wp;
  std::atomic<int64_t> next(0);
  auto worker = [&]() {
    std::vector<RawPoint> raw;
    for (;;) {
      int64_t c = next.fetch_add(1);
      if (c >= num_clouds) break;
      raw.clear();
      for (int f = 0; f < frames_per_cloud; ++f) {
        uint64_t fid = (first_cloud_id + (uint64_t)c) * 64 + (uint64_t)f;
        scan(w, frame_poses + (c * frames_per_cloud + f) * 12, origin_poses + c * 12, rings,
             azimuths, max_range, sigma, seed, fid, &raw);
      }
      counts[c] = finish_cloud(raw, ds_res, n_target, seed, first_cloud_id + (uint64_t)c,
                               order_random, mu + c * n_target * 3, cov + c * n_target * 6,
                               nrm + c * n_target * 3);
    }
  };
  if (num_threads < 1) num_threads = 1;
  std::vector<std::thread> pool;
  for (int i = 0; i < num_threads; ++i) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
}

}  // extern "C"
