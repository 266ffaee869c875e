"""Bench of the on-device registration loop (gvox_register_batch; SURVEY §8(f)
NEXT-1) on the odometry configs of BASELINE.json:

  C2  one 20k-point frame vs 10 keyframe maps (validation on, r = 0.25/0.5/1 m)
  C3  30 frames x 10 keyframe factors x 20k points: 30 independent problems

Keyframe poses at ground truth (fixed), frame poses at the perturbed
linearization points (5 cm / 0.5 deg).  Per config: device time of the loop
graph (CUDA events around the one graph launch, GVOX_TIMER_REGISTER), the
host wall time of the whole call (H2D, graph build + launch, D2H), the
iterations, and point-factor linearizations per second; the oracle loop
(oracle/register.py, all host cores) timed once as the CPU baseline.
Prints one JSON line per config.

Usage: python tools/bench_register.py [--reps 20] [--configs C2,C3] [--no-oracle]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--configs", default="C2,C3")
    ap.add_argument("--max-iterations", type=int, default=10)
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--no-oracle", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2407_10344_b200 as gv
    ctx = gv.Context(0)
    for name in a.configs.split(","):
        sc = synth.make(name)
        variable = sorted(set(int(v) for v in sc.factors[:, 2]))
        poses = sc.gt_poses.copy()
        poses[variable] = sc.poses[variable]
        clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
        maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
        kw = dict(max_iterations=a.max_iterations, eps_rot=a.eps, eps_trans=a.eps)
        for _ in range(3):
            gv.register_batch(ctx, clouds, maps, sc.factors, poses, **kw)
        torch.cuda.synchronize()
        ctx.enable_timing(True)
        ctx.timing(reset=True)
        gv.launch_count(reset=True)
        t0 = time.perf_counter()
        for _ in range(a.reps):
            p, r, _ = gv.register_batch(ctx, clouds, maps, sc.factors, poses, **kw)
        wall = (time.perf_counter() - t0) / a.reps
        tm = ctx.timing(reset=True)
        ctx.enable_timing(False)
        dev_ms = tm["register"][0] / max(tm["register"][1], 1)
        it = r["iterations"][variable]
        pf_per_iter = sc.point_factors
        # every loop iteration re-linearizes all factors (converged problems
        # stay in the batch until the last one stops)
        loop_iters = int(it.max())
        Tg = sc.gt_poses[variable].reshape(-1, 3, 4)
        Tp = p[variable].reshape(-1, 3, 4)
        T0 = poses[variable].reshape(-1, 3, 4)
        line = {
            "metric": "registrations/s (on-device Gauss-Newton loop)",
            "config": name, "problems": len(variable), "factors": int(len(sc.factors)),
            "point_factors_per_iteration": pf_per_iter,
            "iterations_max": loop_iters, "iterations_mean": float(it.mean()),
            "status": {str(k): int(v) for k, v in zip(*np.unique(r["status"][variable], return_counts=True))},
            "device_ms_per_call": dev_ms,
            "device_us_per_iteration": 1e3 * dev_ms / loop_iters,
            "wall_ms_per_call": 1e3 * wall,
            "registrations_per_s_device": len(variable) / (dev_ms * 1e-3),
            "registrations_per_s_wall": len(variable) / wall,
            "point_factors_per_s_device": pf_per_iter * loop_iters / (dev_ms * 1e-3),
            "launches_per_call": gv.launch_count(reset=True) / a.reps,
            "trans_err_m": {"start_mean": float(np.linalg.norm(T0[:, :, 3] - Tg[:, :, 3], axis=1).mean()),
                            "end_mean": float(np.linalg.norm(Tp[:, :, 3] - Tg[:, :, 3], axis=1).mean())},
        }
        if not a.no_oracle:
            from oracle import oracle as oo
            from oracle import register as oreg
            ocl = [sc.cloud(c) for c in range(sc.num_clouds)]
            omp = [oo.VoxelMap(*sc.cloud(int(c))[:2], sc.r0, sc.levels) for c in sc.map_clouds]
            threads = len(os.sched_getaffinity(0))
            t0 = time.perf_counter()
            op, orr, _ = oreg.register_batch(ocl, omp, sc.factors, poses, num_threads=threads, **kw)
            osec = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": len(variable) / osec, "unit": "registrations/s",
                                    "cores": threads, "kind": "oracle", "seconds": osec,
                                    "sample": f"the whole {name} registration (all problems)"}
            line["oracle_max_trans_diff_m"] = float(np.abs(op[variable, 3::4] - p[variable, 3::4]).max())
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
