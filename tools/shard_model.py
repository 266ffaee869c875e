"""Shard timing model of the factor-sharded C5 step on ONE B200 (
VERDICT r01 item 4): every rank's share of the step -- S1 build of its target
maps, S2 screening of its candidate pairs, S3-S7 linearization of its selected
factors, exactly bench.py's per-rank step -- is timed alone on the one GPU for
N = 2, 4, 8 under two balancing rules (dist.target_weights on candidates only,
and on the previous step's screening decisions).  Predicted strong-scaling
efficiency = T_1 / (N * (max_r T_r + t_gather)), t_gather an estimate of one
NCCL all_gather of the compact records over NVLink (stated in the output).

    python tools/shard_model.py [--submaps M] > gpurun_out/shard_model.json
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--submaps", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import paper_2407_10344_b200 as gv
    from paper_2407_10344_b200 import dist as gdist
    import synth

    kw = {"n_submaps": args.submaps} if args.submaps else {}
    t0 = time.perf_counter()
    sc = synth.make("C5", **kw)
    gen_s = time.perf_counter() - t0
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = gv.Context(0, stream)
    clouds = gv.create_clouds(ctx, torch.from_numpy(sc.mu).to(dev), torch.from_numpy(sc.cov).to(dev),
                              torch.from_numpy(sc.nrm).to(dev), sc.offsets)
    carr = gv.HandleArray(clouds)
    poses = gv.as_poses(sc.poses)
    n_pts = np.diff(sc.offsets)

    def shard_step(targets, pairs_local, all_fac, sel_d, acc, sel_h):
        maps = gv.create_voxelmaps(ctx, [clouds[int(sc.map_clouds[t])] for t in targets], sc.r0,
                                   sc.levels)
        marr = gv.HandleArray(maps)
        if len(pairs_local):
            gv.overlap_select(ctx, carr, marr, pairs_local, poses, sc.overlap_level, 1, 20, out=sel_d)
            ns = gv.linearize_batch_accum_select(ctx, carr, marr, all_fac, sel_d, poses, acc,
                                                 selected_host=sel_h)
        else:
            ns = 0
        return maps, ns

    def time_shard(bounds, r):
        lo, hi = bounds[r], bounds[r + 1]
        rows, loc = gdist.local_pairs(sc.pairs, bounds, r)
        targets = np.arange(lo, hi)
        pl = gv.as_pairs(loc)
        all_fac = np.zeros(len(loc), gv.FACTOR_DTYPE)
        for i, name in enumerate(("source_cloud", "target_map", "pose_i", "pose_j")):
            all_fac[name] = loc[:, i]
        sel_d = torch.empty(max(len(loc), 1), dtype=torch.uint8, device=dev)
        acc = gv.device_records(ctx, max(len(loc), 1), gv.FACTOR_ACCUM_DTYPE)
        sel_h = np.zeros(len(loc), np.uint8)
        shard_step(targets, pl, all_fac, sel_d, acc, sel_h)  # warm-up
        ms = []
        ns = 0
        for _ in range(args.reps):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            maps, ns = shard_step(targets, pl, all_fac, sel_d, acc, sel_h)
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            del maps
        sel_g = np.zeros(len(sc.pairs), bool)
        sel_g[rows] = sel_h.astype(bool)
        return statistics.median(ms), ns, int(n_pts[loc[sel_h.astype(bool), 0]].sum()), sel_g

    M = len(sc.map_clouds)
    t1, nf1, pf1, sel = time_shard([0, M], 0)
    rec_bytes = 288
    out = {"workload": f"C5: {M} submaps x {int(n_pts.mean())} points, {len(sc.pairs)} candidate pairs",
           "generated_s": gen_s, "reps": args.reps,
           "single_gpu": {"ms": t1, "factors": nf1, "point_factors": pf1},
           "t_gather_model": "one NCCL all_gather_into_tensor of (fmax + 1) x 288 B per rank over "
                             "NVLink 5 / NVSwitch: bytes / 400 GB/s effective + 30 us latency "
                             "(an estimate; never measured: the pool has one GPU per call)",
           "modes": {}}
    for mode in ("candidates", "selected"):
        res = {}
        for N in (2, 4, 8):
            w = gdist.target_weights(n_pts, sc.map_clouds, sc.pairs,
                                     sel if mode == "selected" else None)
            b = gdist.shard_targets(n_pts, sc.map_clouds, sc.pairs, N, weights=w)
            ts, nfs = [], []
            for r in range(N):
                t, nf, _, _ = time_shard(b, r)
                ts.append(t)
                nfs.append(nf)
            fmax = max(len(gdist.local_pairs(sc.pairs, b, r)[0]) for r in range(N))
            gbytes = N * (fmax + 1) * rec_bytes
            t_g = 1e3 * (gbytes / 400e9) + 0.03
            tN = max(ts) + t_g
            res[str(N)] = {"bounds": b, "rank_ms": ts, "rank_factors": nfs,
                           "max_ms": max(ts), "mean_ms": statistics.mean(ts),
                           "imbalance_max_over_mean": max(ts) / statistics.mean(ts),
                           "t_gather_ms_est": t_g, "predicted_step_ms": tN,
                           "predicted_efficiency": t1 / (N * tN),
                           "sum_rank_ms_over_single": sum(ts) / t1}
            print(mode, N, json.dumps(res[str(N)]), file=sys.stderr, flush=True)
        out["modes"][mode] = res
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
