"""Small-size driver of the kernels added beyond the §8(a) hot path, for
compute-sanitizer (memcheck / racecheck / synccheck):
  python tools/sanitize_next.py            (plain run: also checks results are sane)
  compute-sanitizer --tool memcheck python tools/sanitize_next.py
Covers: FAST linearize on hash maps with validation, gvox_register_batch (graph
WHILE loop), gvox_overlap_union (> 32 members), gvox_knn / covariances (batch
with empty, 1-point and short clouds; k = 10 and 20), gvox_solve_global
(persistent PCG and the WHILE-node PCG), gvox_optimize_global."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    import paper_2407_10344_b200 as gv
    ctx = gv.Context(0)
    # odometry-like scene: hash-level maps, validation on
    sc = synth.smoother_window(n_frames=3, n_kf=4, per_frame=2, n_points=3000, rings=32, az=256)
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    lin = gv.linearize_batch(ctx, clouds, maps, sc.factors, sc.poses)
    assert np.isfinite(lin["error"]).all() and lin["inliers"].sum() > 0
    poses = sc.gt_poses.copy()
    poses[:3] = sc.poses[:3]
    p, r, h = gv.register_batch(ctx, clouds, maps, sc.factors, poses, max_iterations=4, history=True)
    assert (r["status"][:3] > 0).all()
    # union overlap with 40 members (two shared-memory chunks)
    allmaps = gv.create_voxelmaps(ctx, clouds, sc.r0, sc.levels)
    members = [[m % len(allmaps), m % len(allmaps)] for m in range(40)]
    cnt = gv.overlap_union(ctx, clouds, allmaps, [[0, 0, 0, 40], [1, 1, 5, 3], [2, 2, 0, 0]], members,
                           sc.gt_poses, 1)
    assert cnt[0] > 0 and cnt[2] == 0
    # k-NN batch with edge cases
    rs = np.random.default_rng(0)
    parts = [sc.cloud(0)[0][:1500], np.zeros((0, 3), np.float32), np.float32([[1, 2, 3]]),
             rs.uniform(-1, 1, (7, 3)).astype(np.float32)]
    pts = np.concatenate(parts)
    off = np.cumsum([0] + [len(x) for x in parts])
    for k in (10, 20):
        nb = gv.knn(ctx, pts, k=k, cell_size=1.0, offsets=off)
        cov, nrm = gv.estimate_covariances(ctx, pts, nb, offsets=off)
        assert np.isfinite(cov).all()
    # global solve / optimize on a small submap graph
    gs = synth.global_scene(n_submaps=6, n_points=8000, half_blocks=2, factor_dist=40.0, cand_dist=60.0)
    f = gs.factors.copy()
    f[:, 4] = 0
    gcl = [gv.Cloud(ctx, *gs.cloud(c)) for c in range(gs.num_clouds)]
    gmp = gv.create_voxelmaps(ctx, [gcl[int(c)] for c in gs.map_clouds], gs.r0, gs.levels)
    fixed = np.zeros(len(gs.poses), np.uint8)
    fixed[0] = 1
    acc = gv.linearize_batch_accum(ctx, gcl, gmp, f, gs.poses)
    d1, r1, _, _ = gv.solve_global(ctx, f, acc, gs.poses, fixed, tol=1e-10, max_iterations=500)
    if not os.environ.get("SAN_NO_GRAPHS"):
        os.environ["GVOX_PCG_GRAPH"] = "1"
        d2, r2, _, _ = gv.solve_global(ctx, f, acc, gs.poses, fixed, tol=1e-10, max_iterations=500)
        del os.environ["GVOX_PCG_GRAPH"]
        assert np.linalg.norm(d1 - d2) <= 1e-6 * max(np.linalg.norm(d1), 1e-30)
    out, res, hist = gv.optimize_global(ctx, gcl, gmp, f, gs.poses, fixed, max_iterations=3)
    assert np.isfinite(out).all()
    print("sanitize_next: ok")


if __name__ == "__main__":
    main()
