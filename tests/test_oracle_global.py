"""Pins of the global Gauss-Newton step oracle (oracle/global_solve.py;
SURVEY §8(f) NEXT-4), CPU only:

* gauge null space: with no pose fixed, moving every pose by the same world
  motion changes no relative pose, so H [Ad(T_v^-1) xi]_v = 0 for every xi
  (a mis-scattered block, a transposed H_ij or a sign error breaks it);
* with one pose fixed the step is a descent step: the total error of the
  graph after T_v <- T_v Exp(delta_v) is below the error before, and the
  poses move toward the ground truth;
* a two-pose graph with the target fixed reduces to the registration step
  -H_ii^-1 b_i (pinned by Kabsch in test_oracle_register.py).
"""
import numpy as np
import pytest

import synth
from oracle import global_solve as og
from tests.se3 import adjoint, right_perturb, to12, to44


@pytest.fixture(scope="module")
def graph(oracle):
    sc = synth.global_scene(n_submaps=8, n_points=20000, half_blocks=2, factor_dist=40.0,
                            cand_dist=60.0)
    clouds = [sc.cloud(c) for c in range(sc.num_clouds)]
    maps = [oracle.VoxelMap(*sc.cloud(int(c))[:2], sc.r0, sc.levels) for c in sc.map_clouds]
    f = sc.factors.copy()
    f[:, 4] = 0
    return sc, clouds, maps, f


def total_error(oracle, clouds, maps, f, poses):
    return sum(d["e"] for d in oracle.linearize_batch(clouds, maps, f, poses, num_threads=8))


def test_gauge_null_space(oracle, graph):
    sc, clouds, maps, f = graph
    lin = oracle.linearize_batch(clouds, maps, f, sc.poses, num_threads=8)
    P = len(sc.poses)
    H, b, var = og.assemble(f, lin, P, np.zeros(P, bool))
    rs = np.random.default_rng(0)
    for _ in range(3):
        xi = rs.normal(0, 1, 6)
        d = np.concatenate([adjoint(to12(np.linalg.inv(to44(sc.poses[v])))) @ xi for v in range(P)])
        assert np.linalg.norm(H @ d) <= 1e-9 * np.linalg.norm(H) * np.linalg.norm(d)
    # and the gradient is orthogonal to the gauge directions (e is invariant)
    assert abs(b @ d) <= 1e-9 * np.linalg.norm(b) * np.linalg.norm(d)


def test_step_descends(oracle, graph):
    sc, clouds, maps, f = graph
    P = len(sc.poses)
    fixed = np.zeros(P, bool)
    fixed[0] = True
    poses = sc.poses.copy()
    poses[0] = sc.gt_poses[0]
    lin = oracle.linearize_batch(clouds, maps, f, poses, num_threads=8)
    H, b, var = og.assemble(f, lin, P, fixed)
    x = og.solve(H, b)
    new = poses.copy()
    for v in range(P):
        if var[v] >= 0:
            new[v] = right_perturb(poses[v], x[6 * var[v]: 6 * var[v] + 6])
    e0 = total_error(oracle, clouds, maps, f, poses)
    e1 = total_error(oracle, clouds, maps, f, new)
    assert e1 < 0.9 * e0
    dt0 = np.linalg.norm(poses[1:, 3::4] - sc.gt_poses[1:, 3::4], axis=1).mean()
    dt1 = np.linalg.norm(new[1:, 3::4] - sc.gt_poses[1:, 3::4], axis=1).mean()
    assert dt1 < 0.5 * dt0


def test_two_pose_graph_is_registration_step(oracle, graph):
    sc, clouds, maps, f = graph
    row = f[:1]
    lin = oracle.linearize_batch(clouds, maps, row, sc.poses, num_threads=4)
    P = len(sc.poses)
    fixed = np.ones(P, bool)
    fixed[row[0, 2]] = False
    H, b, var = og.assemble(row, lin, P, fixed)
    np.testing.assert_array_equal(H, lin[0]["H_ii"])
    np.testing.assert_allclose(og.solve(H, b), -np.linalg.solve(lin[0]["H_ii"], lin[0]["b_i"]),
                               rtol=1e-12, atol=1e-15)


def test_optimize_converges_to_ground_truth(oracle, graph):
    """The loop's fixed point: the graph error drops (GN on a re-linearized,
    re-associated objective is not strictly monotone near the optimum:
    allow 1e-5 relative wobble per step) and the poses end close to the ground
    truth they were perturbed from."""
    sc, clouds, maps, f = graph
    P = len(sc.poses)
    fixed = np.zeros(P, bool)
    fixed[0] = True
    poses = sc.poses.copy()
    poses[0] = sc.gt_poses[0]
    out, errs, conv = og.optimize(clouds, maps, f, poses, fixed, max_iterations=8, eps_rot=1e-7,
                                  eps_trans=1e-6, num_threads=8)
    assert conv
    assert all(b <= a * (1 + 1e-5) for a, b in zip(errs, errs[1:]))
    assert errs[-1] < 0.1 * errs[0]
    dt = np.linalg.norm(out[1:, 3::4] - sc.gt_poses[1:, 3::4], axis=1)
    dt0 = np.linalg.norm(poses[1:, 3::4] - sc.gt_poses[1:, 3::4], axis=1)
    assert dt.mean() < 0.2 * dt0.mean() and dt.max() < 0.02
