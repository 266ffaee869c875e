// oracle.cpp -- plain, slow, fp64 CPU oracle of the VGICP hot path of
// GLIM (arXiv 2407.10344).  TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
// --impl reference) may load this library.  The product path
// (paper_2407_10344_b200/, libgvox.so) never includes, links or calls it, and
// this file includes nothing from the product tree: the two share no code,
// headers, tables or constants.
//
// Citations: "P:n" = /root/reference/PAPER.md line n (Sec. III-C "Matching
// Cost Factor": Preprocessing P:186, Correspondence search P:197,
// Linearization P:199-218 with Eq.2, Eq.3, Eqs.4-8
// P:213-218; overlap rate P:280, global factor threshold P:391).  "S:n" =
// SPEC.md line n.  Readings of ambiguous passages are the numbered readings
// Q1..Q19 of SURVEY.md Sec.8(c); DESIGN.md lists every one.
//
// Every function evaluates its definition directly, in fp64, with no blocking,
// fusion or reordering: per level an ordered std::map keyed by the packed voxel
// key, per point the 3x12 Jacobian J = [A | B], the full 12x12 J^T Omega J, and
// an independent (Cholesky) inverse of the fused covariance.  The adjoint
// shortcut used by the GPU path is deliberately NOT used here.
//
// Compiled with -O2 -ffp-contract=off (no fast-math) so that every a*b+c is
// two roundings unless written as std::fma.  The few std::fma chains below are
// the pinned operation orders of reading Q10 (discrete decisions: voxel keys
// and the visibility test must be reproducible bit for bit).
//
// Parity pins (tests/test_oracle_*.py, -m "not gpu"): brute-force binning and
// containing-cell scans, the e = 1/2 worked value, exact zero error and
// gradient at ground truth on a dyadic lattice, central finite differences of
// e versus 2b, the gauge null space and adjoint identities, left-invariance,
// level additivity, and Gauss-Newton recovery of a known displacement.

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <thread>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// Voxel keys.  P:197: "q_k = floor(p_k / r)".  P:186: "the voxel size of the
// l-th voxelmap is given by r^l = r0 2^(l-1)"; 0-based here, r_l = r0 * 2^l
// (Q14).  Packed key (Q11): 21 bits per axis, each axis offset by 2^20.
// ---------------------------------------------------------------------------
const int64_t kKeyHalf = int64_t(1) << 20;

bool key_in_range(int64_t k) { return k >= -kKeyHalf && k < kKeyHalf; }

uint64_t pack_key(int64_t kx, int64_t ky, int64_t kz) {
  return (uint64_t(kx + kKeyHalf) << 42) | (uint64_t(ky + kKeyHalf) << 21) |
         uint64_t(kz + kKeyHalf);
}

double level_resolution(double r0, int level) { return std::ldexp(r0, level); }

// floor(x / r) with a correctly rounded fp64 division (Q10).
int64_t voxel_coord(double x, double r) { return (int64_t)std::floor(x / r); }

// ---------------------------------------------------------------------------
// Poses: 3x4 row-major [R | t], world <- sensor.  T_ij = T_j^-1 T_i maps
// source-frame (P_i) points into the target frame (P_j) -- reading Q1/R1.
// Pinned fma order of Q10.
// ---------------------------------------------------------------------------
struct Pose {
  double R[3][3];
  double t[3];
};

Pose load_pose(const double* T) {
  Pose p;
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) p.R[a][b] = T[a * 4 + b];
    p.t[a] = T[a * 4 + 3];
  }
  return p;
}

// T_ij = T_j^-1 T_i  (R_ij = R_j^T R_i, t_ij = R_j^T (t_i - t_j)), and the
// viewpoint v = T_i^-1 t_j = R_i^T (t_j - t_i) used by the visibility test of
// P:197.
void relative_pose(const Pose& Ti, const Pose& Tj, Pose* Tij, double v[3]) {
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      Tij->R[a][b] = std::fma(Tj.R[0][a], Ti.R[0][b],
                              std::fma(Tj.R[1][a], Ti.R[1][b], Tj.R[2][a] * Ti.R[2][b]));
  double dt[3] = {Ti.t[0] - Tj.t[0], Ti.t[1] - Tj.t[1], Ti.t[2] - Tj.t[2]};
  for (int a = 0; a < 3; ++a)
    Tij->t[a] = std::fma(Tj.R[0][a], dt[0], std::fma(Tj.R[1][a], dt[1], Tj.R[2][a] * dt[2]));
  double dv[3] = {Tj.t[0] - Ti.t[0], Tj.t[1] - Ti.t[1], Tj.t[2] - Ti.t[2]};
  for (int a = 0; a < 3; ++a)
    v[a] = std::fma(Ti.R[0][a], dv[0], std::fma(Ti.R[1][a], dv[1], Ti.R[2][a] * dv[2]));
}

// q = R mu + t, pinned order q_a = fma(R_a0, x, fma(R_a1, y, fma(R_a2, z, t_a))).
void transform_point(const Pose& T, const double mu[3], double q[3]) {
  for (int a = 0; a < 3; ++a)
    q[a] = std::fma(T.R[a][0], mu[0], std::fma(T.R[a][1], mu[1], std::fma(T.R[a][2], mu[2], T.t[a])));
}

// P:197 visibility: discard if (p_k - T_i^-1 t_j) . n_k > 0 (strict, Q7).
// Pinned order: fma(dx, nx, fma(dy, ny, dz * nz)).
bool is_invisible(const double mu[3], const double n[3], const double v[3]) {
  double dx = mu[0] - v[0], dy = mu[1] - v[1], dz = mu[2] - v[2];
  double dot = std::fma(dx, n[0], std::fma(dy, n[1], dz * n[2]));
  return dot > 0.0;
}

// ---------------------------------------------------------------------------
// Voxelmap: "we create a sparse voxelmap with spatial voxel hashing and
// take the average of the points and their covariances in each voxel".
// Per voxel: arithmetic mean of member means, arithmetic mean of member
// covariances (Q9), member count.  Canonical order = ascending packed key.
// ---------------------------------------------------------------------------
struct Acc {
  double sum_mu[3] = {0, 0, 0};
  double sum_cov[6] = {0, 0, 0, 0, 0, 0};  // xx xy xz yy yz zz
  int64_t count = 0;
};

struct Voxel {
  double mean[3];
  double cov[3][3];
  int64_t count;
};

}  // namespace

struct OracleMap {
  double r0 = 0;
  int levels = 0;
  std::vector<std::map<uint64_t, Voxel>> level;  // [levels]
};

namespace {

const Voxel* find_voxel(const OracleMap* m, int level, const double q[3]) {
  double r = level_resolution(m->r0, level);
  int64_t kx = voxel_coord(q[0], r), ky = voxel_coord(q[1], r), kz = voxel_coord(q[2], r);
  if (!key_in_range(kx) || !key_in_range(ky) || !key_in_range(kz)) return nullptr;
  auto it = m->level[level].find(pack_key(kx, ky, kz));
  if (it == m->level[level].end()) return nullptr;
  return &it->second;
}

// Inverse of a symmetric positive-definite 3x3 matrix by Cholesky
// factorisation C = L L^T, then Omega = L^-T L^-1.  Returns false when C is not
// positive definite (Q16: the term is skipped and counted as degenerate).
bool spd_inverse(const double C[3][3], double Omega[3][3]) {
  double L[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j <= i; ++j) {
      double s = C[i][j];
      for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
      if (i == j) {
        if (!(s > 0.0) || !std::isfinite(s)) return false;
        L[i][i] = std::sqrt(s);
      } else {
        L[i][j] = s / L[j][j];
      }
    }
  }
  // Linv = L^-1 (lower triangular) by forward substitution on the identity.
  double Li[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int c = 0; c < 3; ++c) {
    for (int i = 0; i < 3; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= L[i][k] * Li[k][c];
      Li[i][c] = s / L[i][i];
    }
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += Li[k][i] * Li[k][j];
      Omega[i][j] = s;
    }
  return true;
}

void hat(const double w[3], double S[3][3]) {
  S[0][0] = 0;     S[0][1] = -w[2]; S[0][2] = w[1];
  S[1][0] = w[2];  S[1][1] = 0;     S[1][2] = -w[0];
  S[2][0] = -w[1]; S[2][1] = w[0];  S[2][2] = 0;
}

void load_cov(const float* c6, double C[3][3]) {
  C[0][0] = c6[0]; C[0][1] = c6[1]; C[0][2] = c6[2];
  C[1][0] = c6[1]; C[1][1] = c6[3]; C[1][2] = c6[4];
  C[2][0] = c6[2]; C[2][1] = c6[4]; C[2][2] = c6[5];
}

}  // namespace

// ===========================================================================
// extern "C" API (ctypes: oracle/oracle.py)
// ===========================================================================
extern "C" {

// Result of one factor, full 12x12 form over (x_i, x_j), rotation-first
// tangents [w_i, rho_i, w_j, rho_j] (right perturbation T <- T Exp(xi)).
struct OracleFactor {
  double H[144];      // sum_k J^T Omega J      (Eqs.6-7 as blocks [[Hii,Hij],[Hij^T,Hjj]])
  double b[12];       // sum_k J^T Omega d      (Eq.8, sign as printed, Q4)
  double e;           // sum_k d^T Omega d      (Eq.2 with Eq.3, no 1/2, Q4)
  double H_abs[144];  // sum_k |J^T Omega J| elementwise (tolerance denominators, Q13)
  double b_abs[12];   // sum_k |J^T Omega d| elementwise
  int32_t inliers[8];     // hits per level
  int64_t num_invisible;  // points discarded by the P:197 test
  int64_t num_degenerate; // (point, level) terms skipped: fused covariance not PD (Q16)
};

// Returns a new map or NULL with *status = 1 (a key outside +-2^20, the
// GVOX_ERR_RANGE case) / 2 (bad arguments).
OracleMap* oracle_build_voxelmap(const float* mu, const float* cov, int64_t n, double r0,
                                 int levels, int* status) {
  *status = 0;
  if (!(r0 > 0.0) || !std::isfinite(r0) || levels < 1 || levels > 8 || n < 0) {
    *status = 2;
    return nullptr;
  }
  OracleMap* m = new OracleMap;
  m->r0 = r0;
  m->levels = levels;
  m->level.resize(levels);
  for (int l = 0; l < levels; ++l) {
    double r = level_resolution(r0, l);
    std::map<uint64_t, Acc> acc;
    for (int64_t i = 0; i < n; ++i) {
      double x = mu[3 * i + 0], y = mu[3 * i + 1], z = mu[3 * i + 2];
      int64_t kx = voxel_coord(x, r), ky = voxel_coord(y, r), kz = voxel_coord(z, r);
      if (!key_in_range(kx) || !key_in_range(ky) || !key_in_range(kz)) {
        delete m;
        *status = 1;
        return nullptr;
      }
      Acc& a = acc[pack_key(kx, ky, kz)];
      a.sum_mu[0] += x;
      a.sum_mu[1] += y;
      a.sum_mu[2] += z;
      for (int c = 0; c < 6; ++c) a.sum_cov[c] += (double)cov[6 * i + c];
      a.count += 1;
    }
    for (auto& kv : acc) {
      const Acc& a = kv.second;
      Voxel v;
      for (int c = 0; c < 3; ++c) v.mean[c] = a.sum_mu[c] / (double)a.count;
      double c6[6];
      for (int c = 0; c < 6; ++c) c6[c] = a.sum_cov[c] / (double)a.count;
      v.cov[0][0] = c6[0]; v.cov[0][1] = c6[1]; v.cov[0][2] = c6[2];
      v.cov[1][0] = c6[1]; v.cov[1][1] = c6[3]; v.cov[1][2] = c6[4];
      v.cov[2][0] = c6[2]; v.cov[2][1] = c6[4]; v.cov[2][2] = c6[5];
      v.count = a.count;
      m->level[l].emplace(kv.first, v);
    }
  }
  return m;
}

void oracle_map_free(OracleMap* m) { delete m; }

int64_t oracle_map_num_voxels(const OracleMap* m, int level) {
  return (int64_t)m->level[level].size();
}

// Canonical (ascending key) export.  means [V*3], covs [V*6] (xx xy xz yy yz zz).
void oracle_map_export(const OracleMap* m, int level, int64_t* keys, double* means, double* covs,
                       int64_t* counts) {
  int64_t i = 0;
  for (const auto& kv : m->level[level]) {
    keys[i] = (int64_t)kv.first;
    for (int c = 0; c < 3; ++c) means[3 * i + c] = kv.second.mean[c];
    const double(*C)[3] = kv.second.cov;
    double c6[6] = {C[0][0], C[0][1], C[0][2], C[1][1], C[1][2], C[2][2]};
    for (int c = 0; c < 6; ++c) covs[6 * i + c] = c6[c];
    counts[i] = kv.second.count;
    ++i;
  }
}

// Packed key of the voxel containing q at `level`, or -1 if absent
// (no neighbour search, Q8).
int64_t oracle_lookup(const OracleMap* m, int level, const double* q) {
  double r = level_resolution(m->r0, level);
  int64_t kx = voxel_coord(q[0], r), ky = voxel_coord(q[1], r), kz = voxel_coord(q[2], r);
  if (!key_in_range(kx) || !key_in_range(ky) || !key_in_range(kz)) return -1;
  uint64_t key = pack_key(kx, ky, kz);
  return m->level[level].count(key) ? (int64_t)key : -1;
}

int64_t oracle_pack_key(int64_t kx, int64_t ky, int64_t kz) { return (int64_t)pack_key(kx, ky, kz); }

void oracle_relative_pose(const double* Ti, const double* Tj, double* Tij_out, double* v_out) {
  Pose pi = load_pose(Ti), pj = load_pose(Tj), pij;
  relative_pose(pi, pj, &pij, v_out);
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) Tij_out[a * 4 + b] = pij.R[a][b];
    Tij_out[a * 4 + 3] = pij.t[a];
  }
}

// Overlap: number of points of P_i (frame i) that fall within a voxel
// of P_j at `level`, with the relative pose T_ij = T_j^-1 T_i.  No validation
// (Q15).  The rate is count / n (0 for an empty source).
int64_t oracle_overlap(const float* mu, int64_t n, const OracleMap* m, const double* Ti,
                       const double* Tj, int level) {
  Pose pi = load_pose(Ti), pj = load_pose(Tj), T;
  double v[3];
  relative_pose(pi, pj, &T, v);
  int64_t count = 0;
  for (int64_t k = 0; k < n; ++k) {
    double p[3] = {mu[3 * k], mu[3 * k + 1], mu[3 * k + 2]}, q[3];
    transform_point(T, p, q);
    if (find_voxel(m, level, q)) ++count;
  }
  return count;
}

// One matching cost factor, evaluated at the linearization point
// (T_i, T_j).  If eval_Ti/eval_Tj are non-NULL, correspondences and Omega are
// taken at (T_i, T_j) (Omega "fixed at the linearization point") but the
// residuals d_k and Jacobians at (eval_Ti, eval_Tj) -- used by the
// finite-difference pins.  corr (optional, [n][levels]) receives the packed key
// of the corresponding voxel, -1 for none, -2 for a point discarded by the
// visibility test.
void oracle_linearize(const float* mu, const float* cov, const float* normals, int64_t n,
                      const OracleMap* m, const double* Ti, const double* Tj, int validate,
                      const double* eval_Ti, const double* eval_Tj, OracleFactor* out,
                      int64_t* corr) {
  std::memset(out, 0, sizeof(OracleFactor));
  Pose pi = load_pose(Ti), pj = load_pose(Tj), T, Te;
  double v[3], ve[3];
  relative_pose(pi, pj, &T, v);
  if (eval_Ti && eval_Tj) {
    Pose ei = load_pose(eval_Ti), ej = load_pose(eval_Tj);
    relative_pose(ei, ej, &Te, ve);
  } else {
    Te = T;
  }
  const int L = m->levels;
  for (int64_t k = 0; k < n; ++k) {
    double p[3] = {mu[3 * k], mu[3 * k + 1], mu[3 * k + 2]};
    if (validate && normals) {
      double nk[3] = {normals[3 * k], normals[3 * k + 1], normals[3 * k + 2]};
      bool has_normal = !(nk[0] == 0.0 && nk[1] == 0.0 && nk[2] == 0.0);
      if (has_normal && is_invisible(p, nk, v)) {
        out->num_invisible += 1;
        if (corr)
          for (int l = 0; l < L; ++l) corr[k * L + l] = -2;
        continue;
      }
    }
    double q[3], qe[3];
    transform_point(T, p, q);   // correspondence search at the linearization point
    transform_point(Te, p, qe); // residual / Jacobian evaluation point
    double Ck[3][3];
    load_cov(cov + 6 * k, Ck);
    // T_ij C_k T_ij^T = R C_k R^T (Q6), at the linearization point.
    double RC[3][3], RCRt[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0;
        for (int c = 0; c < 3; ++c) s += T.R[a][c] * Ck[c][b];
        RC[a][b] = s;
      }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0;
        for (int c = 0; c < 3; ++c) s += RC[a][c] * T.R[b][c];
        RCRt[a][b] = s;
      }
    for (int l = 0; l < L; ++l) {
      const Voxel* vox = find_voxel(m, l, q);
      if (corr) {
        if (vox) {
          double r = level_resolution(m->r0, l);
          corr[k * L + l] = (int64_t)pack_key(voxel_coord(q[0], r), voxel_coord(q[1], r),
                                               voxel_coord(q[2], r));
        } else {
          corr[k * L + l] = -1;
        }
      }
      if (!vox) continue;
      // Eq.3: Omega_k = (C~ + T_ij C_k T_ij^T)^-1, fixed at the linearization point.
      double Cf[3][3], Om[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) Cf[a][b] = vox->cov[a][b] + RCRt[a][b];
      if (!spd_inverse(Cf, Om)) {
        out->num_degenerate += 1;
        continue;
      }
      // d_k = mu~ - T_ij mu_k (Eq.3 text).
      double d[3] = {vox->mean[0] - qe[0], vox->mean[1] - qe[1], vox->mean[2] - qe[2]};
      // Eq.4: A_k = [R_ij (mu_k)x, -R_ij];  Eq.5: B_k = [-(T_ij mu_k)x, I] (Q3).
      double Sm[3][3], Sq[3][3];
      hat(p, Sm);
      hat(qe, Sq);
      double J[3][12];
      for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) {
          double s = 0;
          for (int c = 0; c < 3; ++c) s += Te.R[a][c] * Sm[c][b];
          J[a][b] = s;                        // R (mu)x
          J[a][3 + b] = -Te.R[a][b];          // -R
          J[a][6 + b] = -Sq[a][b];            // -(q)x
          J[a][9 + b] = (a == b) ? 1.0 : 0.0; // I
        }
      }
      // Eqs.6-8 as the full 12x12 J^T Omega J and 12-vector J^T Omega d (Q2).
      double OJ[3][12], Od[3];
      for (int a = 0; a < 3; ++a) {
        for (int c = 0; c < 12; ++c) {
          double s = 0;
          for (int b = 0; b < 3; ++b) s += Om[a][b] * J[b][c];
          OJ[a][c] = s;
        }
        double s = 0;
        for (int b = 0; b < 3; ++b) s += Om[a][b] * d[b];
        Od[a] = s;
      }
      for (int r = 0; r < 12; ++r) {
        for (int c = 0; c < 12; ++c) {
          double s = 0;
          for (int a = 0; a < 3; ++a) s += J[a][r] * OJ[a][c];
          out->H[r * 12 + c] += s;
          out->H_abs[r * 12 + c] += std::fabs(s);
        }
        double s = 0;
        for (int a = 0; a < 3; ++a) s += J[a][r] * Od[a];
        out->b[r] += s;
        out->b_abs[r] += std::fabs(s);
      }
      double e = 0;
      for (int a = 0; a < 3; ++a) e += d[a] * Od[a];
      out->e += e;  // Eq.2: sum over levels and points
      out->inliers[l] += 1;
    }
  }
}

// Batch of factors on a std::thread pool (one thread per requested core).
// factors: [F][5] int64 {source cloud, target map, pose i, pose j, flags};
// flags bit0 = validate surface.  poses [P][12].
void oracle_linearize_batch(const float* const* mus, const float* const* covs,
                            const float* const* normals, const int64_t* npts,
                            const OracleMap* const* maps, const int64_t* factors,
                            int64_t num_factors, const double* poses, int num_threads,
                            OracleFactor* out) {
  std::atomic<int64_t> next(0);
  auto worker = [&]() {
    for (;;) {
      int64_t f = next.fetch_add(1);
      if (f >= num_factors) break;
      const int64_t* fr = factors + 5 * f;
      int64_t s = fr[0], t = fr[1];
      oracle_linearize(mus[s], covs[s], normals[s], npts[s], maps[t], poses + 12 * fr[2],
                       poses + 12 * fr[3], (int)(fr[4] & 1), nullptr, nullptr, out + f, nullptr);
    }
  };
  if (num_threads < 1) num_threads = 1;
  std::vector<std::thread> pool;
  for (int i = 0; i < num_threads; ++i) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
}

// Overlap counts for a batch of pairs {source cloud, target map, pose i, pose j}.
void oracle_overlap_batch(const float* const* mus, const int64_t* npts,
                          const OracleMap* const* maps, const int64_t* pairs, int64_t num_pairs,
                          const double* poses, int level, int num_threads, int64_t* counts) {
  std::atomic<int64_t> next(0);
  auto worker = [&]() {
    for (;;) {
      int64_t p = next.fetch_add(1);
      if (p >= num_pairs) break;
      const int64_t* pr = pairs + 4 * p;
      counts[p] = oracle_overlap(mus[pr[0]], npts[pr[0]], maps[pr[1]], poses + 12 * pr[2],
                                 poses + 12 * pr[3], level);
    }
  };
  if (num_threads < 1) num_threads = 1;
  std::vector<std::thread> pool;
  for (int i = 0; i < num_threads; ++i) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
}

// P:280 "the overlap rate between that frame and the union of all keyframes":
// the number of points of the source (at pose Ti) whose key at `level` is
// occupied in at least one of the K maps (map k at pose Tjs + 12 k).
int64_t oracle_overlap_union(const float* mu, int64_t n, const OracleMap* const* maps,
                             const double* Tjs, int64_t K, const double* Ti, int level) {
  std::vector<Pose> T(K);
  Pose pi = load_pose(Ti);
  for (int64_t j = 0; j < K; ++j) {
    double v[3];
    relative_pose(pi, load_pose(Tjs + 12 * j), &T[j], v);
  }
  int64_t count = 0;
  for (int64_t k = 0; k < n; ++k) {
    double p[3] = {mu[3 * k], mu[3 * k + 1], mu[3 * k + 2]};
    bool hit = false;
    for (int64_t j = 0; j < K && !hit; ++j) {
      double q[3];
      transform_point(T[j], p, q);
      hit = find_voxel(maps[j], level, q) != nullptr;
    }
    if (hit) ++count;
  }
  return count;
}

int oracle_sizeof_factor(void) { return (int)sizeof(OracleFactor); }

}  // extern "C"
