"""Pins of the oracle's matching cost factor (Eqs. 2-8), CPU only.

Pins (each independent of the oracle's own formulas):
* worked value e = 1/2 for unit covariances, d = (1,0,0), T = I;
* exact zero error and gradient at ground truth on a dyadic lattice where all
  fp arithmetic is exact (SURVEY Sec.8c "Zero at ground truth");
* central finite differences of e (Omega, correspondences frozen) in
  the right-perturbation tangent of T_i and T_j equal 2b (reading Q4);
* at zero residual the FD Hessian of e equals 2H (Gauss-Newton is exact there);
* gauge null space H [xi; Ad(T_ij) xi] = 0 and b_i = -Ad^T b_j (the relative
  pose is invariant to a common motion);
* left-invariance under a common world motion, level additivity (Eq.2 sums
  levels), visibility examples of S:256-258 (Fig.3);
* Gauss-Newton on H_ii, b_i recovers the Kabsch/Umeyama alignment (textbook
  special case with isotropic covariances, one point per voxel).
"""
import numpy as np
import pytest

from tests.se3 import (adjoint, plane_cov, random_pose, rel_pose, right_perturb, se3_exp, to12,
                       to44)

I12 = to12(np.eye(4))
UNIT = np.array([1, 0, 0, 1, 0, 1], np.float32)


def scene(rs, n=400, noise=0.02, r0=0.5, L=3, extent=6.0):
    """Structured scene: points on a few planes, plane-like covariances; the
    target is the source seen from another pose plus noise."""
    normals = np.array([[0, 0, 1], [1, 0, 0], [0, 1, 0], [0.6, 0.8, 0]], float)
    pts, covs, nrms = [], [], []
    for k in range(n):
        nv = normals[k % 4]
        t1 = np.cross(nv, [0.3, 0.5, 0.7]); t1 /= np.linalg.norm(t1)
        t2 = np.cross(nv, t1)
        p = nv * (k % 4) * 0.7 + t1 * rs.uniform(-extent, extent) + t2 * rs.uniform(-extent, extent)
        pts.append(p)
        covs.append(plane_cov(nv))
        nrms.append(nv)
    return (np.array(pts, np.float32), np.array(covs, np.float32), np.array(nrms, np.float32))


def make_pair(rs, oracle, n=400, noise=0.02, r0=0.5, L=3, pose_noise=(0.02, 0.05)):
    mu_w, cov_w, n_w = scene(rs, n)
    Ti = random_pose(rs, 0.5, 3.0)
    Tj = random_pose(rs, 0.5, 3.0)
    # source in frame i, target in frame j (both observe the same world points)
    Ti44, Tj44 = to44(Ti), to44(Tj)
    src = (mu_w.astype(float) - Ti44[:3, 3]) @ Ti44[:3, :3]
    tgt = (mu_w.astype(float) - Tj44[:3, 3]) @ Tj44[:3, :3] + rs.normal(0, noise, (n, 3))
    def rot_cov(c6, R):
        out = []
        for c in c6:
            C = np.array([[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]], float)
            C = R.T @ C @ R
            out.append([C[0, 0], C[0, 1], C[0, 2], C[1, 1], C[1, 2], C[2, 2]])
        return np.array(out, np.float32)
    src_cov = rot_cov(cov_w, Ti44[:3, :3])
    tgt_cov = rot_cov(cov_w, Tj44[:3, :3])
    src_n = (n_w @ Ti44[:3, :3]).astype(np.float32)
    m = oracle.VoxelMap(tgt.astype(np.float32), tgt_cov, r0, L)
    # linearization point: perturb T_i slightly
    Ti_lin = right_perturb(Ti, np.concatenate([rs.normal(0, pose_noise[0], 3),
                                               rs.normal(0, pose_noise[1], 3)]))
    return src.astype(np.float32), src_cov, src_n, m, Ti_lin, Tj


def test_worked_value_half(oracle):
    # isotropic unit covariances, d = (1,0,0), T_ij = I -> e = 1/2.
    m = oracle.VoxelMap(np.array([[3.5, 1.0, 1.0]], np.float32), UNIT[None], 4.0, 1)
    src = np.array([[2.5, 1.0, 1.0]], np.float32)
    r = oracle.linearize(src, UNIT[None], None, m, I12, I12)
    # (the Cholesky inverse of 2I is 1/2 up to one rounding of 1/sqrt(2)^2)
    assert r["e"] == pytest.approx(0.5, rel=1e-15)
    assert r["inliers"].tolist() == [1]
    # b_j translation part = Omega d = (1/2, 0, 0); rotation part = q x Omega d
    np.testing.assert_allclose(r["b_j"][3:], [0.5, 0, 0], rtol=1e-15, atol=0)
    np.testing.assert_allclose(r["b_j"][:3], np.cross([2.5, 1.0, 1.0], [0.5, 0, 0]), rtol=1e-15, atol=0)
    np.testing.assert_allclose(r["H_jj"][3:, 3:], 0.5 * np.eye(3), rtol=1e-15, atol=0)


def test_worked_value_rotated_anisotropic(oracle):
    # Eq.3 with a rotation: C_k = diag(1, 3, 0.5), T_ij = Rz(90 deg) so
    # T_ij C_k T_ij^T = diag(3, 1, 0.5); C~ = I; d = (1, 0, 0)
    # -> e = 1 / (1 + 3) = 1/4 (hand computation, Q6: rotation acts, translation not).
    Rz = np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1.0]])
    Ti = np.eye(4); Ti[:3, :3] = Rz; Ti[:3, 3] = [0.0, 0.0, 0.0]
    q = np.array([2.5, 1.0, 1.0])
    src = (Rz.T @ q)[None].astype(np.float32)
    m = oracle.VoxelMap(np.array([[3.5, 1.0, 1.0]], np.float32), UNIT[None], 4.0, 1)
    cs = np.array([[1, 0, 0, 3, 0, 0.5]], np.float32)
    r = oracle.linearize(src, cs, None, m, to12(Ti), I12)
    assert r["e"] == pytest.approx(0.25, rel=1e-15)
    # and with d along z: e = 1 / (1 + 0.5)
    m2 = oracle.VoxelMap(np.array([[2.5, 1.0, 2.0]], np.float32), UNIT[None], 4.0, 1)
    r2 = oracle.linearize(src, cs, None, m2, to12(Ti), I12)
    assert r2["e"] == pytest.approx(1 / 1.5, rel=1e-15)


def test_zero_error_and_gradient_at_ground_truth_lattice(oracle):
    # points on a 8 m lattice (alone in their voxel at r = 1, 2, 4), dyadic
    # coordinates, 90-degree rotations and dyadic translations: every fp op exact.
    g = np.stack(np.meshgrid(np.arange(-2, 3), np.arange(-2, 3), np.arange(0, 2),
                             indexing="ij"), -1).reshape(-1, 3)
    src = (g * 8.0 + np.array([1.5, 2.25, 3.125])).astype(np.float32)
    Rz = np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1.0]])
    Rx = np.array([[1, 0, 0], [0, 0, -1], [0, 1, 0.0]])
    Ti = np.eye(4); Ti[:3, :3] = Rz; Ti[:3, 3] = [16.0, -8.0, 0.0]
    Tj = np.eye(4); Tj[:3, :3] = Rx; Tj[:3, 3] = [-24.0, 8.0, 32.0]
    Tij = np.linalg.inv(Tj) @ Ti
    tgt = (src.astype(float) @ Tij[:3, :3].T + Tij[:3, 3]).astype(np.float32)
    assert np.all(tgt.astype(float) == src.astype(float) @ Tij[:3, :3].T + Tij[:3, 3])
    cov = np.tile(np.array(plane_cov([0.3, 0.4, 0.866]), np.float32), (len(src), 1))
    m = oracle.VoxelMap(tgt, cov, 1.0, 3)
    for l in range(3):
        assert m.num_voxels(l) == len(src)
    r = oracle.linearize(src, cov, None, m, to12(Ti), to12(Tj))
    assert r["inliers"].tolist() == [len(src)] * 3
    assert r["e"] == 0.0
    assert np.all(r["b"] == 0.0)
    H = r["H"]
    w = np.linalg.eigvalsh(0.5 * (H + H.T))
    assert w.min() >= -1e-9 * w.max()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gradient_is_half_fd_of_error(oracle, seed):
    rs = np.random.default_rng(seed)
    src, cov, nrm, m, Ti, Tj = make_pair(rs, oracle)
    r = oracle.linearize(src, cov, None, m, Ti, Tj)
    assert r["inliers"].sum() > 100
    h = 1e-6
    g = np.zeros(12)
    for k in range(12):
        xi = np.zeros(6)
        xi[k % 6] = h
        if k < 6:
            ep = oracle.linearize(src, cov, None, m, Ti, Tj, eval_Ti=right_perturb(Ti, xi), eval_Tj=Tj)
            em = oracle.linearize(src, cov, None, m, Ti, Tj, eval_Ti=right_perturb(Ti, -xi), eval_Tj=Tj)
        else:
            ep = oracle.linearize(src, cov, None, m, Ti, Tj, eval_Ti=Ti, eval_Tj=right_perturb(Tj, xi))
            em = oracle.linearize(src, cov, None, m, Ti, Tj, eval_Ti=Ti, eval_Tj=right_perturb(Tj, -xi))
        g[k] = (ep["e"] - em["e"]) / (2 * h)
    # Reading Q4: e(delta) ~ e + 2 b^T delta + delta^T H delta
    err = np.linalg.norm(g - 2 * r["b"]) / np.linalg.norm(2 * r["b"])
    assert err < 1e-5, err


def test_fd_hessian_equals_2H_at_zero_residual(oracle):
    # each source point alone in its voxel (8 m lattice, r = 1); target =
    # fp32(T_ij mu), so d is fp32 rounding only and GN's H is the exact Hessian/2
    rs = np.random.default_rng(3)
    g = np.stack(np.meshgrid(np.arange(-2, 3), np.arange(-2, 3), np.arange(0, 2),
                             indexing="ij"), -1).reshape(-1, 3)
    src = (g * 8.0 + rs.uniform(2, 6, g.shape)).astype(np.float32)
    cov = np.array([plane_cov(rs.normal(0, 1, 3)) for _ in range(len(src))], np.float32)
    Ti = random_pose(rs, 0.5, 3.0)
    Tj = random_pose(rs, 0.5, 3.0)
    Tij = to44(rel_pose(Ti, Tj))
    tgt = (src.astype(float) @ Tij[:3, :3].T + Tij[:3, 3]).astype(np.float32)
    m = oracle.VoxelMap(tgt, cov, 1.0, 1)
    r = oracle.linearize(src, cov, None, m, Ti, Tj)
    assert r["inliers"][0] == len(src)
    h = 1e-4
    Hfd = np.zeros((12, 12))

    def e_at(xi12):
        return oracle.linearize(src, cov, None, m, Ti, Tj, eval_Ti=right_perturb(Ti, xi12[:6]),
                                eval_Tj=right_perturb(Tj, xi12[6:]))["e"]
    for a in range(12):
        for b in range(a, 12):
            ea = np.zeros(12); ea[a] = h
            eb = np.zeros(12); eb[b] = h
            v = (e_at(ea + eb) - e_at(ea - eb) - e_at(-ea + eb) + e_at(-ea - eb)) / (4 * h * h)
            Hfd[a, b] = Hfd[b, a] = v
    err = np.linalg.norm(Hfd - 2 * r["H"]) / np.linalg.norm(2 * r["H"])
    assert err < 1e-4, err


@pytest.mark.parametrize("seed", [4, 5])
def test_gauge_null_space_and_adjoint_identities(oracle, seed):
    rs = np.random.default_rng(seed)
    src, cov, nrm, m, Ti, Tj = make_pair(rs, oracle)
    r = oracle.linearize(src, cov, None, m, Ti, Tj)
    Ad = adjoint(rel_pose(Ti, Tj))
    H = r["H"]
    for _ in range(4):
        xi = rs.normal(0, 1, 6)
        v = np.concatenate([xi, Ad @ xi])
        assert np.linalg.norm(H @ v) <= 1e-12 * np.linalg.norm(H) * np.linalg.norm(v) * 100
    scale = np.abs(r["H"]).max()
    np.testing.assert_allclose(r["b_i"], -Ad.T @ r["b_j"], rtol=0, atol=1e-10 * max(1, np.abs(r["b_abs"]).max()))
    np.testing.assert_allclose(r["H_ii"], Ad.T @ r["H_jj"] @ Ad, rtol=0, atol=1e-10 * scale)
    np.testing.assert_allclose(r["H_ij"], -Ad.T @ r["H_jj"], rtol=0, atol=1e-10 * scale)
    # symmetric, PSD, exactly 6 (numerically) zero eigenvalues
    np.testing.assert_allclose(H, H.T, rtol=0, atol=1e-12 * scale)
    w = np.linalg.eigvalsh(0.5 * (H + H.T))
    assert w.min() >= -1e-9 * w.max()
    assert np.sum(w < 1e-9 * w.max()) == 6


def test_left_invariance(oracle):
    rs = np.random.default_rng(8)
    src, cov, nrm, m, Ti, Tj = make_pair(rs, oracle)
    G = to44(random_pose(rs, 1.0, 20.0))
    r0 = oracle.linearize(src, cov, None, m, Ti, Tj, return_corr=True)
    r1 = oracle.linearize(src, cov, None, m, to12(G @ to44(Ti)), to12(G @ to44(Tj)),
                          return_corr=True)
    assert np.array_equal(r0["corr"], r1["corr"])
    np.testing.assert_allclose(r1["e"], r0["e"], rtol=1e-9)
    np.testing.assert_allclose(r1["H"], r0["H"], rtol=0, atol=1e-9 * np.abs(r0["H"]).max())
    np.testing.assert_allclose(r1["b"], r0["b"], rtol=0, atol=1e-9 * np.abs(r0["b_abs"]).max())


def test_level_additivity(oracle):
    rs = np.random.default_rng(9)
    src, cov, nrm, m, Ti, Tj = make_pair(rs, oracle, r0=0.5, L=3)
    r = oracle.linearize(src, cov, None, m, Ti, Tj)
    mu_t, cov_t = m.mu, m.cov
    e_sum, b_sum, H_sum = 0.0, np.zeros(12), np.zeros((12, 12))
    for l in range(3):
        ml = oracle.VoxelMap(mu_t, cov_t, 0.5 * 2 ** l, 1)
        rl = oracle.linearize(src, cov, None, ml, Ti, Tj)
        assert rl["inliers"][0] == r["inliers"][l]
        e_sum += rl["e"]; b_sum += rl["b"]; H_sum += rl["H"]
    np.testing.assert_allclose(e_sum, r["e"], rtol=1e-12)
    np.testing.assert_allclose(b_sum, r["b"], rtol=0, atol=1e-10 * np.abs(r["b_abs"]).max())
    np.testing.assert_allclose(H_sum, r["H"], rtol=0, atol=1e-10 * np.abs(r["H"]).max())


def test_visibility_examples(oracle):
    # S:256-257 / Fig.3: wall at x = 0 with normal (-1,0,0); viewer at x = -1
    # sees it, viewer at x = +1 does not.  Frame i = identity; the target map is
    # the same wall point expressed in frame j (so it always corresponds).
    mu = np.array([[0.0, 0.3, 0.2]], np.float32)
    nrm = np.array([[-1.0, 0.0, 0.0]], np.float32)

    def run(x, normals=nrm):
        Tj = to44(I12)
        Tj[0, 3] = x
        m = oracle.VoxelMap(mu - np.array([[x, 0, 0]], np.float32), UNIT[None], 1.0, 1)
        return oracle.linearize(mu, UNIT[None], normals, m, I12, to12(Tj), validate=True,
                                return_corr=True)
    r = run(-1.0)
    assert r["num_invisible"] == 0 and r["inliers"][0] == 1
    r = run(1.0)
    assert r["num_invisible"] == 1 and r["inliers"][0] == 0 and r["corr"][0, 0] == -2
    assert r["e"] == 0.0
    # sign-crossing sweep: invisible exactly when viewer x > 0 (strict)
    for x in [-0.5, -1e-6, 0.0, 1e-6, 0.5]:
        assert run(x)["num_invisible"] == int(x > 0)
    # zero normal = no validation (Q7)
    assert run(1.0, np.zeros((1, 3), np.float32))["num_invisible"] == 0


def test_empty_overlap_and_degenerate(oracle):
    rs = np.random.default_rng(10)
    src, cov, nrm, m, Ti, Tj = make_pair(rs, oracle)
    far = to44(Ti)
    far[:3, 3] += 1000.0
    r = oracle.linearize(src, cov, None, m, to12(far), Tj)
    assert r["e"] == 0.0 and np.all(r["H"] == 0) and r["inliers"].sum() == 0
    # exactly-zero covariances: fused covariance singular -> term skipped (Q16)
    z = np.zeros((1, 6), np.float32)
    m0 = oracle.VoxelMap(np.array([[0.5, 0.5, 0.5]], np.float32), z, 1.0, 1)
    r = oracle.linearize(np.array([[0.2, 0.5, 0.5]], np.float32), z, None, m0, I12, I12)
    assert r["num_degenerate"] == 1 and r["inliers"][0] == 0 and r["e"] == 0.0


def test_batch_equals_serial(oracle):
    rs = np.random.default_rng(12)
    clouds, maps, poses = [], [], [I12]
    factors = []
    for f in range(6):
        src, cov, nrm, m, Ti, Tj = make_pair(rs, oracle, n=150)
        clouds.append((src, cov, nrm))
        maps.append(m)
        poses += [Ti, Tj]
        factors.append([f, f, 1 + 2 * f, 2 + 2 * f, f % 2])
    out = oracle.linearize_batch(clouds, maps, factors, np.array(poses), num_threads=3)
    for f, (s, c, n) in enumerate(clouds):
        r = oracle.linearize(s, c, n, maps[f], poses[1 + 2 * f], poses[2 + 2 * f], validate=bool(f % 2))
        assert out[f]["e"] == r["e"]
        assert np.array_equal(out[f]["H"], r["H"]) and np.array_equal(out[f]["b"], r["b"])


def test_gauss_newton_recovers_kabsch(oracle):
    # Isotropic equal covariances, one point per voxel, exact correspondences:
    # GN with delta_i = -H_ii^-1 b_i, T_i <- T_i Exp(delta_i) converges to the
    # least-squares (Kabsch/Umeyama) alignment.
    rs = np.random.default_rng(13)
    g = np.stack(np.meshgrid(np.arange(-3, 3), np.arange(-3, 3), np.arange(0, 3),
                             indexing="ij"), -1).reshape(-1, 3)
    tgt = (g * 8.0 + 4.0 + rs.normal(0, 0.05, g.shape)).astype(np.float32)
    cov = np.tile(np.array([0.5, 0, 0, 0.5, 0, 0.5], np.float32), (len(tgt), 1))
    Tj = to12(np.eye(4))
    T_true = se3_exp(np.array([0.05, -0.03, 0.08, 0.3, -0.2, 0.1]))
    src = ((tgt.astype(float) - T_true[:3, 3]) @ T_true[:3, :3] + rs.normal(0, 0.01, g.shape)).astype(np.float32)
    m = oracle.VoxelMap(tgt, cov, 8.0, 1)
    Ti = to12(np.eye(4))
    es = []
    for it in range(8):
        r = oracle.linearize(src, cov, None, m, Ti, Tj)
        assert r["inliers"][0] == len(src)
        es.append(r["e"])
        delta = -np.linalg.solve(r["H_ii"], r["b_i"])
        Ti = right_perturb(Ti, delta)
    assert es[-1] < es[0] * 1e-2
    # Kabsch (SVD) of src -> tgt
    P = src.astype(float); Q = tgt.astype(float)
    pc, qc = P.mean(0), Q.mean(0)
    U, S, Vt = np.linalg.svd((P - pc).T @ (Q - qc))
    D = np.diag([1, 1, np.sign(np.linalg.det(Vt.T @ U.T))])
    R = Vt.T @ D @ U.T
    t = qc - R @ pc
    T = to44(Ti)
    np.testing.assert_allclose(T[:3, :3], R, atol=1e-9)
    np.testing.assert_allclose(T[:3, 3], t, atol=1e-8)
