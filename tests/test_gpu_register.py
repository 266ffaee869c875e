"""On-device registration loop (gvox_register_batch through the C ABI) vs the
oracle loop (oracle/register.py) and vs the Kabsch closed form.

Bars: at the first linearization (same pose on both sides) inliers are
bit-exact and e within 1e-5 (tests/parity.py); one step's pose agrees to
1e-4 of the step (H, b within 1e-4, so delta = -H^-1 b within ~1e-4); the
converged pose agrees to 2e-5 m / 2e-6 rad (a fixed point of the loop:
H/b differences of 1e-4 shift it by far less than that on these scenes);
status and iteration counts equal.  Batched problems equal serial runs bit
for bit (fixed summation order, fixed tile plan).
"""
import numpy as np
import pytest
import scipy.linalg

import synth
from oracle import register as oreg
from tests.parity import E_TOL
from tests.se3 import to12, to44

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(gv):
    return gv.Context(0)


@pytest.fixture(scope="module")
def c2():
    return synth.odometry_step(n_kf=10, n_points=20000)


@pytest.fixture(scope="module")
def c3():
    return synth.smoother_window(n_frames=6, n_kf=8, per_frame=4, n_points=8000, rings=64, az=512)


def reg_poses(sc, variable):
    """Fixed poses at ground truth, variable poses at the perturbed point."""
    p = sc.gt_poses.copy()
    for v in variable:
        p[v] = sc.poses[v]
    return p


def gpu_inputs(gv, ctx, sc):
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    return clouds, maps


def oracle_inputs(oracle, sc):
    clouds = [sc.cloud(c) for c in range(sc.num_clouds)]
    maps = [oracle.VoxelMap(*sc.cloud(int(c))[:2], sc.r0, sc.levels) for c in sc.map_clouds]
    return clouds, maps


def rot_angle(Ra, Rb):
    return float(np.linalg.norm(scipy.linalg.logm(Ra.T @ Rb).real)) / np.sqrt(2)


def test_one_step_parity(gv, ctx, oracle, c2):
    sc = c2
    poses = reg_poses(sc, [0])
    g_cl, g_mp = gpu_inputs(gv, ctx, sc)
    o_cl, o_mp = oracle_inputs(oracle, sc)
    for lam in (0.0, 50.0):
        gp, gr, gh = gv.register_batch(ctx, g_cl, g_mp, sc.factors, poses, max_iterations=1,
                                       lam=lam, eps_rot=0, eps_trans=0, history=True)
        op, orr, oh = oreg.register_batch(o_cl, o_mp, sc.factors, poses, max_iterations=1,
                                          lam=lam, eps_rot=0, eps_trans=0, num_threads=8)
        assert gr[0]["inliers"] == orr[0]["inliers"]
        assert gr[0]["status"] == orr[0]["status"] == oreg.REG_MAX_ITER
        assert abs(gr[0]["error_initial"] - orr[0]["error_initial"]) <= E_TOL * orr[0]["error_initial"]
        assert gh[0, 0] == gr[0]["error_initial"]
        step = np.linalg.norm(orr[0]["last_step"])
        assert np.linalg.norm(gr[0]["last_step"] - orr[0]["last_step"]) <= 1e-4 * step
        Tg, To = to44(gp[0]), to44(op[0])
        assert np.linalg.norm(Tg[:3, 3] - To[:3, 3]) <= 1e-4 * step + 1e-9
        assert rot_angle(Tg[:3, :3], To[:3, :3]) <= 1e-4 * step + 1e-9
        np.testing.assert_array_equal(gp[1:], poses[1:])
        assert all(int(gr[j]["status"]) == gv.REG_FIXED for j in range(1, len(poses)))


def test_converged_parity_c2(gv, ctx, oracle, c2):
    sc = c2
    poses = reg_poses(sc, [0])
    g_cl, g_mp = gpu_inputs(gv, ctx, sc)
    o_cl, o_mp = oracle_inputs(oracle, sc)
    kw = dict(max_iterations=20, eps_rot=1e-7, eps_trans=1e-7)
    gp, gr, gh = gv.register_batch(ctx, g_cl, g_mp, sc.factors, poses, history=True, **kw)
    op, orr, oh = oreg.register_batch(o_cl, o_mp, sc.factors, poses, num_threads=8, **kw)
    assert gr[0]["status"] == orr[0]["status"] == oreg.REG_CONVERGED
    assert gr[0]["iterations"] == orr[0]["iterations"]
    n = int(gr[0]["iterations"])
    np.testing.assert_allclose(gh[:n, 0], oh[:n, 0], rtol=1e-4)
    Tg, To = to44(gp[0]), to44(op[0])
    assert np.linalg.norm(Tg[:3, 3] - To[:3, 3]) <= 2e-5
    assert rot_angle(Tg[:3, :3], To[:3, :3]) <= 2e-6
    # and the loop did its job: closer to ground truth than the start
    Tgt, T0 = to44(sc.gt_poses[0]), to44(poses[0])
    assert np.linalg.norm(Tg[:3, 3] - Tgt[:3, 3]) < 0.3 * np.linalg.norm(T0[:3, 3] - Tgt[:3, 3])


def test_batch_equals_serial_and_device_outputs(gv, ctx, oracle, c3):
    sc = c3
    nf = 6
    poses = reg_poses(sc, range(nf))
    g_cl, g_mp = gpu_inputs(gv, ctx, sc)
    kw = dict(max_iterations=8, eps_rot=1e-6, eps_trans=1e-6)
    bp, br, bh = gv.register_batch(ctx, g_cl, g_mp, sc.factors, poses, history=True, **kw)
    for v in range(nf):
        assert int(br[v]["status"]) == gv.REG_CONVERGED
        rows = sc.factors[sc.factors[:, 2] == v]
        sp, sr, sh = gv.register_batch(ctx, g_cl, g_mp, rows, poses, history=True, **kw)
        assert np.array_equal(sp[v], bp[v]), v
        assert sr[v].tobytes() == br[v].tobytes(), v
        assert np.array_equal(sh[:, v], bh[:, v])
    dp, dr, dh = gv.register_batch(ctx, g_cl, g_mp, sc.factors, poses, history=True, device=True,
                                   **kw)
    import torch
    torch.cuda.synchronize()
    assert np.array_equal(dp.cpu().numpy(), bp)
    assert dr.cpu().numpy().tobytes() == br.tobytes()
    assert np.array_equal(dh.cpu().numpy(), bh)
    # the batch matches the oracle loop too
    o_cl, o_mp = oracle_inputs(oracle, sc)
    op, orr, oh = oreg.register_batch(o_cl, o_mp, sc.factors, poses, num_threads=8, **kw)
    for v in range(nf):
        assert int(br[v]["iterations"]) == orr[v]["iterations"], v
        assert np.abs(to44(bp[v])[:3, 3] - to44(op[v])[:3, 3]).max() <= 2e-5


def test_kabsch_closed_form(gv, ctx):
    # textbook case (tests/test_oracle_register.py): the GPU loop lands on the
    # SVD alignment directly, no oracle involved
    rs = np.random.default_rng(13)
    g = np.stack(np.meshgrid(np.arange(-3, 3), np.arange(-3, 3), np.arange(0, 3),
                             indexing="ij"), -1).reshape(-1, 3)
    tgt = (g * 8.0 + 4.0 + rs.normal(0, 0.05, g.shape)).astype(np.float32)
    cov = np.tile(np.array([0.5, 0, 0, 0.5, 0, 0.5], np.float32), (len(tgt), 1))
    T_true = oreg.se3_exp(np.array([0.05, -0.03, 0.08, 0.3, -0.2, 0.1]))
    src = ((tgt.astype(float) - T_true[:3, 3]) @ T_true[:3, :3] +
           rs.normal(0, 0.01, g.shape)).astype(np.float32)
    cs, ct = gv.Cloud(ctx, src, cov), gv.Cloud(ctx, tgt, cov)
    m = gv.create_voxelmap(ctx, ct, 8.0, 1)
    poses = np.stack([to12(np.eye(4)), to12(np.eye(4))])
    p, r, _ = gv.register_batch(ctx, [cs], [m], [[0, 0, 0, 1, 0]], poses, max_iterations=10,
                                eps_rot=1e-6, eps_trans=1e-6)
    P, Q = src.astype(float), tgt.astype(float)
    pc, qc = P.mean(0), Q.mean(0)
    U, S, Vt = np.linalg.svd((P - pc).T @ (Q - qc))
    D = np.diag([1, 1, np.sign(np.linalg.det(Vt.T @ U.T))])
    R = Vt.T @ D @ U.T
    t = qc - R @ pc
    T = to44(p[0])
    # fp32 per-point algebra: the fixed point moves by ~1e-7 relative
    np.testing.assert_allclose(T[:3, :3], R, atol=2e-6)
    np.testing.assert_allclose(T[:3, 3], t, atol=2e-5)
    assert int(r[0]["status"]) == gv.REG_CONVERGED and int(r[0]["inliers"]) == len(src)


def test_singular_fixed_and_errors(gv, ctx):
    rs = np.random.default_rng(5)
    g = np.stack(np.meshgrid(np.arange(-2, 2), np.arange(-2, 2), np.arange(0, 2),
                             indexing="ij"), -1).reshape(-1, 3)
    tgt = (g * 8.0 + 4.0).astype(np.float32)
    cov = np.tile(np.array([0.5, 0, 0, 0.5, 0, 0.5], np.float32), (len(tgt), 1))
    ct = gv.Cloud(ctx, tgt, cov)
    m = gv.create_voxelmap(ctx, ct, 8.0, 1)
    far = to12(np.array([[1, 0, 0, 1e4], [0, 1, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1.0]]))
    I = to12(np.eye(4))
    poses = np.stack([far, I, I])
    p, r, h = gv.register_batch(ctx, [ct], [m], [[0, 0, 0, 1, 0], [0, 0, 2, 1, 0]], poses,
                                max_iterations=5, eps_rot=1.0, eps_trans=1.0, history=True)
    assert int(r[0]["status"]) == gv.REG_SINGULAR and int(r[0]["iterations"]) == 1
    assert np.array_equal(p[0], far) and int(r[0]["inliers"]) == 0
    assert int(r[1]["status"]) == gv.REG_FIXED and np.array_equal(p[1], I)
    assert int(r[2]["status"]) == gv.REG_CONVERGED and int(r[2]["iterations"]) == 1
    assert h[1:].max() == 0.0
    with pytest.raises(gv.GvoxError, match="variable pose"):
        gv.register_batch(ctx, [ct], [m], [[0, 0, 0, 1, 0], [0, 0, 1, 2, 0]], poses)
    with pytest.raises(gv.GvoxError, match="ERROR_ONLY"):
        gv.register_batch(ctx, [ct], [m], [[0, 0, 0, 1, 2]], poses)
    with pytest.raises(gv.GvoxError, match="pose_i == pose_j"):
        gv.register_batch(ctx, [ct], [m], [[0, 0, 1, 1, 0]], poses)
    with pytest.raises(gv.GvoxError, match="max_iterations"):
        gv.register_batch(ctx, [ct], [m], [[0, 0, 0, 1, 0]], poses, max_iterations=0)
    # no factors: poses copied, all fixed
    p, r, _ = gv.register_batch(ctx, [ct], [m], np.zeros((0, 5), np.int64), poses)
    assert np.array_equal(p, poses) and (r["status"] == gv.REG_FIXED).all()
