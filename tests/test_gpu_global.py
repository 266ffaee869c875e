"""gvox_solve_global on the CUDA path.

* assembly parity: the GPU's assembled H and b (from its own compact records)
  against the oracle's dense assembly of its own factors: each 6x6 block
  within 1e-4 of the block's Frobenius norm scale, b within 1e-4 (the
  linearization bars of tests/parity.py carried through a sum);
* solver: the PCG solution against numpy's direct solve of the GPU's own
  (H, b) to 1e-8 relative, converged flag, bitwise repeatability;
* the step itself against the oracle step (1e-3 relative: cond(H) amplifies
  the 1e-6-level H/b differences), device-resident records, error paths.
"""
import numpy as np
import pytest

import synth
from oracle import global_solve as og

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(gv):
    return gv.Context(0)


@pytest.fixture(scope="module")
def graph(gv, ctx, oracle):
    sc = synth.global_scene(n_submaps=12, n_points=20000, half_blocks=2, factor_dist=40.0,
                            cand_dist=60.0)
    f = sc.factors.copy()
    f[:, 4] = 0
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    ocl = [sc.cloud(c) for c in range(sc.num_clouds)]
    omp = [oracle.VoxelMap(*sc.cloud(int(c))[:2], sc.r0, sc.levels) for c in sc.map_clouds]
    poses = sc.poses.copy()
    poses[0] = sc.gt_poses[0]
    acc = gv.linearize_batch_accum(ctx, clouds, maps, f, poses)
    lin = oracle.linearize_batch(ocl, omp, f, poses, num_threads=8)
    return sc, f, poses, acc, lin, clouds, maps


def test_assembly_and_solve_parity(gv, ctx, graph):
    sc, f, poses, acc, lin, clouds, maps = graph
    P = len(poses)
    fixed = np.zeros(P, np.uint8)
    fixed[0] = 1
    delta, res, H, b = gv.solve_global(ctx, f, acc, poses, fixed, tol=1e-12, max_iterations=2000,
                                       dense=True)
    Ho, bo, var = og.assemble(f, lin, P, fixed.astype(bool))
    V = P - 1
    assert res["num_variables"] == V and res["converged"] == 1
    for i in range(V):
        for j in range(V):
            blk, ref = H[6 * i:6 * i + 6, 6 * j:6 * j + 6], Ho[6 * i:6 * i + 6, 6 * j:6 * j + 6]
            scale = max(np.linalg.norm(Ho[6 * i:6 * i + 6, 6 * i:6 * i + 6]), 1e-30)
            assert np.linalg.norm(blk - ref) <= 1e-4 * scale, (i, j)
    assert np.linalg.norm(b - bo) <= 1e-4 * np.linalg.norm(bo)
    # the solver against a direct solve of the same system
    x = np.linalg.solve(H, -b)
    got = delta[1:].reshape(-1)
    assert np.linalg.norm(got - x) <= 1e-8 * np.linalg.norm(x)
    assert not delta[0].any()
    # the step against the oracle's step
    xo = og.solve(Ho, bo)
    assert np.linalg.norm(got - xo) <= 1e-3 * np.linalg.norm(xo)
    # bitwise repeatable
    d2, r2, H2, b2 = gv.solve_global(ctx, f, acc, poses, fixed, tol=1e-12, max_iterations=2000,
                                     dense=True)
    assert np.array_equal(d2, delta) and np.array_equal(H2, H) and r2.tobytes() == res.tobytes()


def test_device_records_and_errors(gv, ctx, graph):
    import torch
    sc, f, poses, acc, lin, clouds, maps = graph
    P = len(poses)
    fixed = np.zeros(P, np.uint8)
    fixed[0] = 1
    dacc = torch.empty((len(f), gv.FACTOR_ACCUM_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
    gv.linearize_batch_accum(ctx, clouds, maps, f, poses, out=dacc)
    dd, dres, _, _ = gv.solve_global(ctx, f, dacc, poses, fixed, tol=1e-12, max_iterations=2000)
    hd, hres, _, _ = gv.solve_global(ctx, f, acc, poses, fixed, tol=1e-12, max_iterations=2000)
    torch.cuda.synchronize()
    assert np.array_equal(dd.cpu().numpy(), hd)
    with pytest.raises(gv.GvoxError, match="gauge"):
        gv.solve_global(ctx, f, acc, poses, np.zeros(P, np.uint8))
    # damping removes the gauge freedom
    d3, r3, _, _ = gv.solve_global(ctx, f, acc, poses, np.zeros(P, np.uint8), lam=1.0,
                                   tol=1e-10, max_iterations=2000)
    assert r3["converged"] == 1 and np.isfinite(d3).all()
    # everything fixed: zero step
    d4, r4, _, _ = gv.solve_global(ctx, f, acc, poses, np.ones(P, np.uint8))
    assert not d4.any() and r4["num_variables"] == 0


def test_persistent_and_graph_pcg_agree(gv, ctx, graph, monkeypatch):
    """The cooperative persistent PCG and the WHILE-node two-kernel PCG run the
    same recurrence (different dot-product partitions): same solution to the
    solver tolerance, same iteration count within one."""
    sc, f, poses, acc, lin, clouds, maps = graph
    P = len(poses)
    fixed = np.zeros(P, np.uint8)
    fixed[0] = 1
    d1, r1, _, _ = gv.solve_global(ctx, f, acc, poses, fixed, tol=1e-12, max_iterations=2000)
    monkeypatch.setenv("GVOX_PCG_GRAPH", "1")
    d2, r2, _, _ = gv.solve_global(ctx, f, acc, poses, fixed, tol=1e-12, max_iterations=2000)
    assert np.linalg.norm(d1 - d2) <= 1e-8 * np.linalg.norm(d1)
    assert abs(int(r1["iterations"]) - int(r2["iterations"])) <= 1


def test_optimize_global_matches_oracle_loop(gv, ctx, oracle, graph):
    """gvox_optimize_global (relinearize -> assemble -> PCG -> update, on the
    device) against the oracle's dense loop: same iteration count, errors per
    iteration within 1e-4, final poses within 1e-4 m / rad (fp32 per-point
    algebra and PCG tolerance move the fixed point by far less)."""
    from oracle import global_solve as og
    sc, f, poses, acc, lin, clouds, maps = graph
    P = len(poses)
    fixed = np.zeros(P, np.uint8)
    fixed[0] = 1
    out, res, hist = gv.optimize_global(ctx, clouds, maps, f, poses, fixed, max_iterations=8,
                                        eps_rot=1e-6, eps_trans=1e-5)
    ocl = [sc.cloud(c) for c in range(sc.num_clouds)]
    omp = [oracle.VoxelMap(*sc.cloud(int(c))[:2], sc.r0, sc.levels) for c in sc.map_clouds]
    op, oerr, oconv = og.optimize(ocl, omp, f, poses, fixed.astype(bool), max_iterations=8,
                                  eps_rot=1e-6, eps_trans=1e-5, num_threads=8)
    assert int(res["converged"]) == 1 and oconv
    assert int(res["iterations"]) == len(oerr)
    np.testing.assert_allclose(hist, oerr, rtol=1e-4)
    assert np.abs(out[:, 3::4] - op[:, 3::4]).max() <= 1e-4
    assert np.abs(out[:, [0, 1, 2, 4, 5, 6, 8, 9, 10]] - op[:, [0, 1, 2, 4, 5, 6, 8, 9, 10]]).max() <= 1e-4
    np.testing.assert_array_equal(out[0], poses[0])  # the fixed pose is untouched
