"""Bench of the keyframe mechanism on the C3
recipe (20k-point frames, 0.25/0.5/1 m, overlap level 1 m):
  * union overlap: one frame against the union of N_odom = 20 keyframes
    (gvox_overlap_union), device time per query and point-lookups/s, and a
    batch of 30 frames x 20 keyframes in one call;
  * the whole KeyframeList driver over a 50-frame sequence (insertion test,
    pair overlaps of a new keyframe, removal rule): wall ms per frame.
CPU baseline: the oracle's union overlap (C++) on one frame.  One JSON line."""
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
    from oracle import oracle as oo
    ctx = gv.Context(0)
    sc = synth.make("C3")  # 30 frames + 20 keyframe clouds
    C = sc.num_clouds
    clouds = gv.create_clouds(ctx, sc.mu, sc.cov, sc.nrm, sc.offsets)
    maps = gv.create_voxelmaps(ctx, clouds, sc.r0, sc.levels)
    lvl = sc.overlap_level
    kf = list(range(30, 50))
    members = [[k, k] for k in kf]
    one = [[0, 0, 0, len(kf)]]
    batch = [[f, f, 0, len(kf)] for f in range(30)]
    reps = 50
    for _ in range(3):
        gv.overlap_union(ctx, clouds, maps, batch, members, sc.gt_poses, lvl)
    torch.cuda.synchronize()
    res = {}
    for name, q in (("one_frame", one), ("30_frames", batch)):
        ctx.enable_timing(True)
        ctx.timing(reset=True)
        t0 = time.perf_counter()
        for _ in range(reps):
            cnt = gv.overlap_union(ctx, clouds, maps, q, members, sc.gt_poses, lvl)
        wall = (time.perf_counter() - t0) / reps
        t = ctx.timing(reset=True)["overlap"]
        ctx.enable_timing(False)
        dev_ms = t[0] / max(t[1], 1)
        pts = int(sum(sc.cloud_size(f) for f, _, _, _ in q))
        res[name] = {"device_us": 1e3 * dev_ms, "wall_us": 1e6 * wall, "queries": len(q),
                     "points": pts, "point_lookups_upper": pts * len(kf),
                     "points_per_s_device": pts / (dev_ms * 1e-3),
                     "overlap_rate_first": float(cnt[0]) / sc.cloud_size(q[0][0])}
    # the whole driver over a 50-frame sequence
    seq = list(range(C - 1, 29, -1)) + list(range(30))
    kl = gv.KeyframeList(ctx, level=lvl, n_odom=20)
    t0 = time.perf_counter()
    ev = [kl.add_frame(f, clouds, maps, sc.gt_poses) for f in seq]
    drv = (time.perf_counter() - t0) / len(seq)
    # CPU baseline: the oracle union overlap of one frame
    omaps = [oo.VoxelMap(*sc.cloud(k)[:2], sc.r0, sc.levels) for k in kf]
    t0 = time.perf_counter()
    oc = oo.overlap_union(sc.cloud(0)[0], omaps, sc.gt_poses[0], np.stack([sc.gt_poses[k] for k in kf]), lvl)
    cpu_s = time.perf_counter() - t0
    assert oc == int(gv.overlap_union(ctx, clouds, maps, one, members, sc.gt_poses, lvl)[0])
    print(json.dumps({"metric": "keyframe union-overlap test (P:280) and keyframe list update",
                      "config": "C3 recipe, N_odom = 20, overlap level %d" % lvl, "union": res,
                      "driver_ms_per_frame": 1e3 * drv, "frames": len(seq),
                      "inserted": int(sum(e[0] for e in ev)), "removed": int(sum(len(e[1]) for e in ev)),
                      "cpu_baseline": {"value": sc.cloud_size(0) / cpu_s, "unit": "points/s (one frame vs 20 keyframes)",
                                       "cores": 1, "kind": "oracle", "sample": "frame 0 vs the 20 keyframes"}}),
          flush=True)


if __name__ == "__main__":
    main()
