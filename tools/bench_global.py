"""Bench of the global Gauss-Newton step (gvox_solve_global, SURVEY §8(f)
NEXT-4) on C4 (500 submaps x 50k points, ~1e4 factors; the paper's global
mapping): device time of the linearization (compact records) and of
the solve (expand + BSR assembly + block-Jacobi PCG to 1e-10), PCG
iterations; CPU baseline = the oracle's dense assembly + LAPACK solve of the
same records (numpy, all host cores).  One JSON line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402


def main():
    import torch
    import paper_2407_10344_b200 as gv
    from oracle import global_solve as og
    ctx = gv.Context(0)
    name = os.environ.get("CONFIG", "C4")
    sc = synth.make(name)
    f = sc.factors.copy()
    f[:, 4] = 0
    poses = sc.poses.copy()
    poses[0] = sc.gt_poses[0]
    P = len(poses)
    fixed = np.zeros(P, np.uint8)
    fixed[0] = 1
    off = sc.offsets
    clouds = gv.create_clouds(ctx, sc.mu, sc.cov, sc.nrm, off)
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    dacc = torch.empty((len(f), gv.FACTOR_ACCUM_DTYPE.itemsize), dtype=torch.uint8, device="cuda")
    reps = int(os.environ.get("REPS", "10"))
    for _ in range(2):
        gv.linearize_batch_accum(ctx, clouds, maps, f, poses, out=dacc)
        d, r, _, _ = gv.solve_global(ctx, f, dacc, poses, fixed, tol=1e-10, max_iterations=5000)
    torch.cuda.synchronize()
    ctx.enable_timing(True)
    ctx.timing(reset=True)
    for _ in range(reps):
        gv.linearize_batch_accum(ctx, clouds, maps, f, poses, out=dacc)
        d, r, _, _ = gv.solve_global(ctx, f, dacc, poses, fixed, tol=1e-10, max_iterations=5000)
    t = ctx.timing(reset=True)
    ctx.enable_timing(False)
    lin_ms = (t["linearize"][0] + t["reduce"][0]) / reps
    solve_ms = t["solve"][0] / reps
    # CPU baseline: dense assembly + LAPACK of the same (expanded) records
    rec = gv.records_to_numpy(gv.expand(ctx, f, poses, dacc, out=gv.device_records(ctx, len(f), gv.LINEAR_FACTOR_DTYPE)))
    lin = [{"H": np.block([[x["H_ii"].reshape(6, 6), x["H_ij"].reshape(6, 6)],
                          [x["H_ij"].reshape(6, 6).T, x["H_jj"].reshape(6, 6)]]),
            "b": np.concatenate([x["b_i"], x["b_j"]])} for x in rec]
    t0 = time.perf_counter()
    H, b, var = og.assemble(f, lin, P, fixed.astype(bool))
    x = og.solve(H, b)
    cpu_s = time.perf_counter() - t0
    # the whole global optimisation (relinearize -> assemble -> PCG -> update)
    # (one untimed run, then the median of 5: a single wall-clock run varied
    # 133-243 ms between otherwise identical boxes)
    walls = []
    for rep in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        opt_poses, opt_res, opt_hist = gv.optimize_global(ctx, clouds, maps, f, poses, fixed,
                                                          max_iterations=15, eps_rot=1e-6, eps_trans=1e-5)
        if rep:
            walls.append(time.perf_counter() - t0)
    opt_s = float(np.median(walls))
    gt = sc.gt_poses
    opt = {"wall_ms": 1e3 * opt_s, "wall_ms_min": 1e3 * min(walls), "runs": len(walls), "iterations": int(opt_res["iterations"]),
           "converged": int(opt_res["converged"]), "pcg_iterations": int(opt_res["pcg_iterations"]),
           "ms_per_iteration": 1e3 * opt_s / max(int(opt_res["iterations"]), 1),
           "error_initial": float(opt_res["error_initial"]), "error_final": float(opt_res["error_final"]),
           "trans_err_m_start": float(np.linalg.norm(poses[:, 3::4] - gt[:, 3::4], axis=1).mean()),
           "trans_err_m_end": float(np.linalg.norm(opt_poses[:, 3::4] - gt[:, 3::4], axis=1).mean())}
    got = d.cpu().numpy() if hasattr(d, "cpu") else d
    err = float(np.linalg.norm(got[1:].reshape(-1) - x) / np.linalg.norm(x))
    print(json.dumps({
        "metric": "global GN step (linearize + assemble + PCG) ms", "config": name,
        "poses": P, "factors": int(len(f)), "point_factors": sc.point_factors,
        "linearize_ms": lin_ms, "solve_ms": solve_ms, "pcg_iterations": int(r["iterations"]),
        "pcg_converged": int(r["converged"]), "blocks": int(r["num_blocks"]),
        "step_ms": lin_ms + solve_ms, "rel_diff_vs_dense_solve": err, "optimize": opt,
        "cpu_baseline": {"value": cpu_s * 1e3, "unit": "ms (dense assemble + LAPACK solve of the same records)",
                         "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
                         "sample": "the whole solve (linearization excluded)"},
    }), flush=True)


if __name__ == "__main__":
    main()
