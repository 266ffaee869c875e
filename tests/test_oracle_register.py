"""Pins of the registration-loop oracle (oracle/register.py; SURVEY §8(f)
NEXT-1: re-linearize every iteration; Omega fixed per iteration),
CPU only.  Each pin is independent of the oracle's own formulas:

* the closed-form SE(3) exponential equals scipy.linalg.expm of the 4x4 twist
  matrix (the exponential's definition), tiny angles included;
* textbook special case: isotropic equal covariances, one point per voxel,
  exact correspondences -> the loop converges to the Kabsch/Umeyama SVD
  alignment (library SVD), with quadratic convergence of the error;
* structured LiDAR-like scene (synth C2 recipe, smaller): the loop recovers
  the ground-truth displacement from a 5 cm / 0.5 deg perturbation and the
  error decreases;
* a variable pose with no correspondence is singular and left unchanged; a
  loose tolerance converges after one step; converged poses stop early.
"""
import numpy as np
import pytest
import scipy.linalg

from oracle import register as reg
from tests.se3 import hat, to12, to44


def test_se3_exp_matches_matrix_exponential():
    rs = np.random.default_rng(3)
    cases = [rs.normal(0, s, 6) for s in (1.0, 0.3, 1e-3)]
    cases += [np.array([1e-6, -2e-6, 3e-7, 0.5, -0.2, 0.1]), np.zeros(6),
              np.array([0.0, 0.0, np.pi - 1e-3, 1.0, 2.0, 3.0])]
    for xi in cases:
        X = np.zeros((4, 4))
        X[:3, :3] = hat(xi[:3])
        X[:3, 3] = xi[3:]
        np.testing.assert_allclose(reg.se3_exp(xi), scipy.linalg.expm(X), atol=1e-13, rtol=0)


def _kabsch(P, Q):
    pc, qc = P.mean(0), Q.mean(0)
    U, S, Vt = np.linalg.svd((P - pc).T @ (Q - qc))
    D = np.diag([1, 1, np.sign(np.linalg.det(Vt.T @ U.T))])
    R = Vt.T @ D @ U.T
    return R, qc - R @ pc


def kabsch_problem(rs, oracle):
    g = np.stack(np.meshgrid(np.arange(-3, 3), np.arange(-3, 3), np.arange(0, 3),
                             indexing="ij"), -1).reshape(-1, 3)
    tgt = (g * 8.0 + 4.0 + rs.normal(0, 0.05, g.shape)).astype(np.float32)
    cov = np.tile(np.array([0.5, 0, 0, 0.5, 0, 0.5], np.float32), (len(tgt), 1))
    T_true = reg.se3_exp(np.array([0.05, -0.03, 0.08, 0.3, -0.2, 0.1]))
    src = ((tgt.astype(float) - T_true[:3, 3]) @ T_true[:3, :3] +
           rs.normal(0, 0.01, g.shape)).astype(np.float32)
    return src, tgt, cov


def test_loop_converges_to_kabsch(oracle):
    rs = np.random.default_rng(13)
    src, tgt, cov = kabsch_problem(rs, oracle)
    m = oracle.VoxelMap(tgt, cov, 8.0, 1)
    poses = np.stack([to12(np.eye(4)), to12(np.eye(4))])
    out, res, hist = reg.register_batch([(src, cov, None)], [m], [[0, 0, 0, 1, 0]], poses,
                                        max_iterations=10, eps_rot=1e-10, eps_trans=1e-10)
    R, t = _kabsch(src.astype(float), tgt.astype(float))
    T = to44(out[0])
    np.testing.assert_allclose(T[:3, :3], R, atol=1e-10)
    np.testing.assert_allclose(T[:3, 3], t, atol=1e-9)
    np.testing.assert_array_equal(out[1], poses[1])  # the fixed pose is untouched
    assert res[0]["status"] == reg.REG_CONVERGED and res[1]["status"] == reg.REG_FIXED
    assert res[0]["inliers"] == len(src)
    e = hist[: res[0]["iterations"], 0]
    # quadratic convergence to the (non-zero, noisy) optimum
    assert e[0] > 10 * e[1] and abs(e[-1] - e[-2]) <= 1e-9 * e[-1]


@pytest.fixture(scope="module")
def small_c2():
    import synth
    return synth.odometry_step(n_kf=3, n_points=5000, rings=64, az=512)


def _scene_inputs(oracle, sc):
    clouds = [sc.cloud(c) for c in range(sc.num_clouds)]
    maps = [oracle.VoxelMap(*sc.cloud(int(c))[:2], sc.r0, sc.levels) for c in sc.map_clouds]
    return clouds, maps


def test_loop_recovers_displacement(oracle, small_c2):
    sc = small_c2
    clouds, maps = _scene_inputs(oracle, sc)
    poses = sc.gt_poses.copy()
    poses[0] = sc.poses[0]  # the frame starts at the perturbed linearization point
    T0, Tg = to44(poses[0]), to44(sc.gt_poses[0])
    d0 = np.linalg.norm(T0[:3, 3] - Tg[:3, 3])
    assert d0 > 0.02
    out, res, hist = reg.register_batch(clouds, maps, sc.factors, poses, max_iterations=15,
                                        eps_rot=1e-5, eps_trans=1e-5, num_threads=4)
    T = to44(out[0])
    dt = np.linalg.norm(T[:3, 3] - Tg[:3, 3])
    dR = np.linalg.norm(scipy.linalg.logm(Tg[:3, :3].T @ T[:3, :3]).real)
    assert dt < 0.2 * d0 and dt < 0.01, (d0, dt)
    assert dR < np.deg2rad(0.1)
    assert res[0]["status"] == reg.REG_CONVERGED
    assert res[0]["error_final"] < res[0]["error_initial"]
    for j in range(1, len(poses)):
        assert res[j]["status"] == reg.REG_FIXED


def test_singular_and_loose_tolerance(oracle):
    rs = np.random.default_rng(5)
    src, tgt, cov = kabsch_problem(rs, oracle)
    m = oracle.VoxelMap(tgt, cov, 8.0, 1)
    far = to12(np.array([[1, 0, 0, 1e4], [0, 1, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1.0]]))
    I = to12(np.eye(4))
    poses = np.stack([far, I, I])
    factors = [[0, 0, 0, 1, 0], [0, 0, 2, 1, 0]]
    out, res, hist = reg.register_batch([(src, cov, None)], [m], factors, poses,
                                        max_iterations=5, eps_rot=1.0, eps_trans=1.0)
    assert res[0]["status"] == reg.REG_SINGULAR and res[0]["iterations"] == 1
    np.testing.assert_array_equal(out[0], far)
    assert res[0]["inliers"] == 0 and res[0]["error_final"] == 0.0
    assert res[2]["status"] == reg.REG_CONVERGED and res[2]["iterations"] == 1
    assert hist[1:, :].max() == 0.0
