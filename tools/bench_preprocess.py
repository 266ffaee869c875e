"""Bench of the GPU preprocessing (gvox_knn + gvox_estimate_covariances,
SURVEY §8(f) NEXT-3): one 20k-point LiDAR frame (the paper's per-frame k-NN,
P:712, 5.7 ms on its CPU) and the C3 batch (30 frames x 20k points), k = 10.
Device time per call (CUDA events, GVOX_TIMER_PREPROCESS) and points/s; the
oracle's brute-force k-NN timed on a sample of rows as the CPU baseline.
Prints one JSON line per workload."""
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
    from oracle import preprocess as pp
    ctx = gv.Context(0)
    sc = synth.make("C3")
    reps = int(os.environ.get("REPS", "20"))
    cell = float(os.environ.get("CELL", "1.5"))
    for name, ncl in (("frame", 1), ("C3-batch", sc.num_clouds)):
        off = sc.offsets[: ncl + 1]
        pts = torch.from_numpy(sc.mu[: off[-1]]).cuda()
        n = int(off[-1])
        for _ in range(3):
            nb = gv.knn(ctx, pts, 10, cell, off)
            gv.estimate_covariances(ctx, pts, nb, off)
        torch.cuda.synchronize()
        ctx.enable_timing(True)
        ctx.timing(reset=True)
        t0 = time.perf_counter()
        for _ in range(reps):
            nb = gv.knn(ctx, pts, 10, cell, off)
        torch.cuda.synchronize()
        wall_knn = (time.perf_counter() - t0) / reps
        tk = ctx.timing(reset=True)["preprocess"]
        for _ in range(reps):
            gv.estimate_covariances(ctx, pts, nb, off)
        tc = ctx.timing(reset=True)["preprocess"]
        ctx.enable_timing(False)
        knn_ms, cov_ms = tk[0] / reps, tc[0] / reps
        # CPU oracle: brute force on 200 rows of the first cloud
        cl = sc.mu[: sc.offsets[1]]
        t0 = time.perf_counter()
        for i in range(200):
            d2 = pp.sq_dist(cl[i], cl)
            np.lexsort((np.arange(len(cl)), d2))[:10]
        per_row = (time.perf_counter() - t0) / 200
        print(json.dumps({
            "metric": "k-NN (k = 10, exact) + covariance points/s", "workload": name, "clouds": ncl, "cell_size": cell,
            "points": n, "knn_device_ms": knn_ms, "knn_wall_ms": 1e3 * wall_knn,
            "cov_device_ms": cov_ms, "points_per_s_device": n / ((knn_ms + cov_ms) * 1e-3),
            "cpu_baseline": {"value": 1.0 / per_row, "unit": "points/s (k-NN rows)", "cores": 1,
                             "kind": "oracle", "sample": "200 brute-force rows of one 20k frame"},
        }), flush=True)


if __name__ == "__main__":
    main()
