#!/usr/bin/env python
"""bench.py -- throughput of the batched VGICP hot path (GLIM, arXiv 2407.10344)
on B200, in the driver's JSON-line contract.

A STEP is one pass of every hot-path row of SURVEY.md Sec.8(a) over the
workload (default C5: 2000 submaps x 100k points):
  S1  gvox_create_voxelmaps  -- multi-resolution voxelmaps of every target submap
  S2  gvox_overlap_select    -- screening decision of every candidate submap pair:
      a pair becomes a factor iff 20 * count > N_src ("exceeds 5 %"), exact,
      each pair stopping as soon as its decision is certain (C1-C3: gvox_overlap counts)
  S3-S7 gvox_linearize_batch(_accum) -- every selected factor, one batch
  (N > 1: factors sharded by target submap; one NCCL all_gather of the compact
   per-factor records)
value = sum over linearized factors of the source point count / step time
(points linearized per second), inputs (clouds, poses, candidate list)
resident in HBM before the timed region.  e2e = the same metric with clouds
uploaded from pinned host memory and full records downloaded every step.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
torchrun launches one rank per GPU (RANK / LOCAL_RANK / WORLD_SIZE from env).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "VGICP source points linearized/s"
UNIT = "points/s"
WORKLOADS = {
    "C5": "C5 large map: 2000 submaps x 100k points (15 frames each), overlap screening of "
          "candidate pairs, overlap-selected factors (~1e5), r = 0.5/1/2 m",
    "C4": "C4 global: 500 submaps x 50k points, overlap-selected factors, r = 0.5/1/2 m",
    "C3": "C3 smoother window: 30 frames x 10 keyframe factors x 20k points, r = 0.25/0.5/1 m",
    "C2": "C2 odometry step: one 20k frame vs 10 keyframe maps, r = 0.25/0.5/1 m",
    "C1": "C1 single factor: 1k-point source vs 1k-point map, r = 1.0 m, L = 1",
}


def workload_label(args, sc):
    """The workload as run: the config's description, with the submap count and
    points per submap taken from the generated scene when --submaps overrides it."""
    lab = WORKLOADS[args.config]
    if args.config in ("C4", "C5") and args.submaps:
        n = np.diff(sc.offsets)
        lab = (f"{args.config} reduced by --submaps: {sc.num_clouds} submaps x "
               f"{int(n.mean())} points, overlap-selected factors, r = 0.5/1/2 m")
    return lab


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=sorted(WORKLOADS),
                    help="workload; the bench line is C5 (the metric's config), the others "
                         "report per-call latency of the small configs")
    ap.add_argument("--submaps", type=int, default=None, help="override the submap count (tests)")
    ap.add_argument("--order", default="morton", choices=["morton", "random"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-mode", default="pipelined", choices=["pipelined", "serial"],
                    help="e2e: step k+1's upload overlapping step k's compute (default; r02p: "
                         "237 ms vs 367 ms serial per C5 step at 5 steps), or each step's "
                         "upload inside it")
    ap.add_argument("--e2e-steps", type=int, default=20,
                    help="e2e steps timed (the first step's upload is never overlapped)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--per-call-runs", type=int, default=20,
                    help="calls timed for SURVEY 8(d)'s per-call metric (median; 0 = skip)")
    ap.add_argument("--linearize-only", action="store_true",
                    help="profiling aid: time only S3-S7 (not a bench line)")
    return ap.parse_args()


# --------------------------------------------------------------------------- scene
def make_scene(args, rank, world, dist):
    """Rank 0 generates (all host cores); other ranks load it from /dev/shm."""
    import synth
    kw = {}
    if args.submaps:
        kw["n_submaps"] = args.submaps
    if args.order == "random":
        kw["order_random"] = True
    if args.config not in ("C4", "C5"):
        kw = {}
    if world == 1:
        return synth.make(args.config, **kw)
    # rank 0 writes one .npy per array to /dev/shm; every rank maps them
    # read-only (shared page cache, no per-rank copies of the 9 GB clouds)
    base = f"/dev/shm/gvox_bench_{args.config}_{args.submaps}_{args.order}_{os.getppid()}"
    names = ("mu", "cov", "nrm", "offsets", "map_clouds", "factors", "poses", "gt_poses", "pairs")
    if rank == 0:
        sc = synth.make(args.config, **kw)
        for k in names:
            np.save(f"{base}_{k}.npy", getattr(sc, k))
        np.save(f"{base}_meta.npy", np.array([sc.r0, sc.levels, sc.overlap_level]))
    dist.barrier()
    arr = {k: np.load(f"{base}_{k}.npy", mmap_mode="r") for k in names}
    meta = np.load(f"{base}_meta.npy")
    sc = synth.Scene(args.config, arr["mu"], arr["cov"], arr["nrm"], np.array(arr["offsets"]),
                     np.array(arr["map_clouds"]), float(meta[0]), int(meta[1]),
                     np.array(arr["factors"]), np.array(arr["poses"]), np.array(arr["gt_poses"]),
                     np.array(arr["pairs"]), int(meta[2]))
    dist.barrier()
    if rank == 0:  # unlink: the mappings stay valid until every rank exits
        for k in names + ("meta",):
            os.unlink(f"{base}_{k}.npy")
    return sc


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, device_index):
        self.device = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        load = [s for s in sm if s > 300] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- oracle legs
def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_sample(sc, select=True, budget_s=12.0, threads=None):
    """The oracle, as it stands, on a bounded sample of the same step: all rows
    (map build, overlap, selection, linearize) for a random subset of target
    maps, so the mix of work matches the full step.  select: C4/C5 factors are
    the candidates with 20 * count > N; otherwise the config's factor list.
    Returns (points, seconds, description, cores)."""
    from oracle import oracle
    import synth
    cores = threads or synth.host_threads()
    n = np.diff(sc.offsets)
    M = len(sc.map_clouds)
    rs = np.random.default_rng(12345)
    order = rs.permutation(M)
    t0 = time.perf_counter()
    pts = 0
    nf = 0
    npairs = 0
    used = []
    for t in order:
        pr = sc.pairs[sc.pairs[:, 1] == t]
        fr = sc.factors[sc.factors[:, 1] == t]
        if len(pr) == 0 and len(fr) == 0:
            continue
        mu_t, cov_t, _ = sc.cloud(int(sc.map_clouds[t]))
        om = oracle.VoxelMap(mu_t, cov_t, sc.r0, sc.levels)                     # S1
        srcs = sorted(set(int(p[0]) for p in pr) | set(int(f[0]) for f in fr))
        idx = {s_: k for k, s_ in enumerate(srcs)}
        pairs = np.array([[idx[int(p[0])], 0, int(p[2]), int(p[3])] for p in pr], np.int64).reshape(-1, 4)
        counts = oracle.overlap_batch([sc.cloud(s_)[0] for s_ in srcs], [om], pairs, sc.poses,
                                      sc.overlap_level, cores)                  # S2
        if select:
            sel = 20 * counts > n[[srcs[int(p[0])] for p in pairs]]
            fac = np.concatenate([pairs[sel], np.zeros((int(sel.sum()), 1), np.int64)], 1)
        else:
            fac = np.array([[idx[int(f[0])], 0, int(f[2]), int(f[3]), int(f[4])] for f in fr],
                           np.int64).reshape(-1, 5)
        if len(fac):
            oracle.linearize_batch([sc.cloud(s_) for s_ in srcs], [om], fac, sc.poses, cores)  # S3-7
        pts += int(n[[srcs[int(f[0])] for f in fac]].sum()) if len(fac) else 0
        nf += len(fac)
        npairs += len(pairs)
        used.append(int(t))
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    desc = (f"{len(used)} of {M} target maps (random, seed 12345) with all their rows: "
            f"{len(used)} map builds, {npairs} overlap pairs, {nf} factors "
            f"({pts} source points)")
    return pts, dt, desc, cores


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sc = make_scene(args, 0, 1, None)
    samples = []
    desc = None
    cores = None
    for i in range(args.warmup + args.steps):
        budget = max(2.0, 120.0 / max(1, args.warmup + args.steps))
        pts, dt, desc, cores = oracle_sample(sc, args.config in ("C4", "C5"), budget_s=budget)
        if i >= args.warmup:
            samples.append((pts, dt))
    tot_p = sum(p for p, _ in samples)
    tot_t = sum(t for _, t in samples)
    value = tot_p / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / len(samples), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_label(args, sc), "oracle_sample": desc},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": desc, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- main
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # GVOX_DIST_BACKEND=gloo (+ GVOX_SAME_DEVICE=1) runs the multi-rank plumbing on a
        # one-GPU box for testing; the product path is NCCL, one GPU per rank
        backend = os.environ.get("GVOX_DIST_BACKEND", "nccl")
        if os.environ.get("GVOX_SAME_DEVICE"):
            local = 0
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    import __graft_entry__
    __graft_entry__.build()
    import paper_2407_10344_b200 as gv

    t_gen = time.perf_counter()
    sc = make_scene(args, rank, world, dist)
    t_gen = time.perf_counter() - t_gen
    # experiments: the candidate list's order (generated sorted by source) --
    # "target" (by target, then source) or "blockN" (N x N blocks of the
    # (source, target) pair matrix, then source, target)
    po = os.environ.get("GVOX_BENCH_PAIR_ORDER")
    if po and po != "source":
        i_, j_ = sc.pairs[:, 0], sc.pairs[:, 1]
        if po == "target":
            perm = np.lexsort((i_, j_))
        else:
            B_ = int(po[5:])
            perm = np.lexsort((j_, i_, j_ // B_, i_ // B_))
        sc.pairs = np.ascontiguousarray(sc.pairs[perm])
    n_pts = np.diff(sc.offsets)
    log(f"[bench r{rank}] scene {sc.name}: {sc.num_clouds} clouds, {len(sc.mu)} points, "
        f"{len(sc.pairs)} candidate pairs, generated in {t_gen:.1f}s")

    # a non-default stream for everything the step enqueues (the legacy default
    # stream would implicitly serialise with the e2e copy stream)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = gv.Context(dev.index, stream)
    # ---- inputs resident in HBM (not timed)
    mu_d = torch.from_numpy(sc.mu).to(dev)
    cov_d = torch.from_numpy(sc.cov).to(dev)
    nrm_d = torch.from_numpy(sc.nrm).to(dev)
    clouds = gv.create_clouds(ctx, mu_d, cov_d, nrm_d, sc.offsets)
    del mu_d, cov_d, nrm_d
    cloud_arr = gv.HandleArray(clouds)
    poses = gv.as_poses(sc.poses)

    from paper_2407_10344_b200 import dist as gdist
    # C4/C5: factors = candidate pairs whose overlap exceeds 5 %, no
    # validation (Q7).  C1-C3: the config's own factor list (odometry factors,
    # validation on); the overlap of their pairs is still screened.
    select = args.config in ("C4", "C5")

    def setup(bounds):
        """This rank's share of the step for a target-range plan."""
        t_lo, t_hi = bounds[rank], bounds[rank + 1]
        my_targets = np.arange(t_lo, t_hi)
        _, my_pairs = gdist.local_pairs(sc.pairs, bounds, rank)  # target -> local map index
        fixed = None
        if not select:
            fm = (sc.factors[:, 1] >= t_lo) & (sc.factors[:, 1] < t_hi)
            fixed = gv.as_factors(sc.factors[fm])
            fixed["target_map"] -= t_lo
        all_fac = np.zeros(len(my_pairs), gv.FACTOR_DTYPE)  # every candidate as a factor
        for i_, name_ in enumerate(("source_cloud", "target_map", "pose_i", "pose_j")):
            all_fac[name_] = my_pairs[:, i_]
        # device buffers reused across steps
        acc_out = gv.device_records(ctx, max(len(my_pairs), len(sc.factors), 1), gv.FACTOR_ACCUM_DTYPE)
        return (my_targets, my_pairs, gv.as_pairs(my_pairs), n_pts[my_pairs[:, 0]],
                [clouds[int(sc.map_clouds[t])] for t in my_targets], fixed, all_fac, acc_out,
                torch.empty(max(len(my_pairs), 1), dtype=torch.int32, device=dev),
                np.zeros(len(my_pairs), np.uint8),
                torch.empty(max(len(my_pairs), 1), dtype=torch.uint8, device=dev))

    # first plan: candidates' work (no decisions yet); at N > 1 it is redone
    # after the first warm-up step on that step's screening decisions
    bounds = gdist.shard_targets(n_pts, sc.map_clouds, sc.pairs, world)
    (my_targets, my_pairs, pairs_s, src_n, my_target_clouds, fixed, all_fac, acc_out, counts_d,
     sel_h, sel_d) = setup(bounds)
    balance = "candidates (no decisions)"

    state = {}

    host_ms = {"build_call": 0.0, "overlap_call": 0.0, "select": 0.0, "linearize_call": 0.0,
               "gather": 0.0}

    def step(timed_maps=None):
        t0 = time.perf_counter()
        maps = gv.create_voxelmaps(ctx, my_target_clouds, sc.r0, sc.levels)        # S1
        marr = gv.HandleArray(maps)
        t1 = time.perf_counter()
        if select:
            # S2 as the screening decision (overlap exceeds 5 %), kept on
            # the device; S3-S7 over the selected candidates, compacted on the
            # device (one 8-byte readback of the batch size, no host round trip
            # of the decisions before the launch)
            gv.overlap_select(ctx, cloud_arr, marr, pairs_s, poses, sc.overlap_level, 1, 20,
                              out=sel_d)
            t2 = time.perf_counter()
            ns = gv.linearize_batch_accum_select(ctx, cloud_arr, marr, all_fac, sel_d, poses,
                                                 acc_out, selected_host=sel_h)
            t3 = time.perf_counter()
            fac = all_fac[sel_h.view(bool)]  # host bookkeeping, overlaps the linearization
            assert len(fac) == ns
            t4 = time.perf_counter()
            dt_sel, dt_lin = t4 - t3, t3 - t2
        else:
            # S2 as overlap counts of the config's pairs, kept on the device
            # (as the C4/C5 decisions are; e2e reads them back), then S3-S7
            gv.overlap(ctx, cloud_arr, marr, pairs_s, poses, sc.overlap_level, out=counts_d)
            t2 = time.perf_counter()
            fac = fixed
            t3 = time.perf_counter()
            gv.linearize_batch_accum(ctx, cloud_arr, marr, fac, poses, out=acc_out[:len(fac)])
            t4 = time.perf_counter()
            dt_sel, dt_lin = t3 - t2, t4 - t3
        host_ms["build_call"] += 1e3 * (t1 - t0)
        host_ms["overlap_call"] += 1e3 * (t2 - t1)
        host_ms["select"] += 1e3 * dt_sel
        host_ms["linearize_call"] += 1e3 * dt_lin
        if world > 1:
            # the one exchange: all-gather of the compact per-factor records
            state["gathered"], _ = gdist.gather_records(acc_out, len(fac), state["fmax"])
        state["maps"] = maps                  # keep alive until the next step replaces them
        state["fac"] = fac
        return int(n_pts[fac["source_cloud"]].sum()), len(fac)

    # ---- warm-up (also re-balances the shards and sizes the gather)
    warm = args.warmup
    if world > 1:
        if select and warm > 0:
            state["fmax"] = gdist.max_count(max(len(my_pairs), 1), dev)
            step()
            warm -= 1
            # the previous step's screening decisions -> global selection vector
            # -> shards balanced on the work actually selected (setup, untimed)
            rows, _ = gdist.local_pairs(sc.pairs, bounds, rank)
            g = torch.zeros(len(sc.pairs), dtype=torch.int32, device=dev)
            g[torch.from_numpy(rows).to(dev)] = torch.from_numpy(sel_h.astype(np.int32)).to(dev)
            dist.all_reduce(g, op=dist.ReduceOp.SUM)
            w = gdist.target_weights(n_pts, sc.map_clouds, sc.pairs, g.cpu().numpy().astype(bool))
            bounds = gdist.shard_targets(n_pts, sc.map_clouds, sc.pairs, world, weights=w)
            (my_targets, my_pairs, pairs_s, src_n, my_target_clouds, fixed, all_fac, acc_out,
             counts_d, sel_h, sel_d) = setup(bounds)
            balance = "previous step's screening decisions (selected point-factors)"
        state["fmax"] = gdist.max_count(max(len(my_pairs), 1), dev)
        acc_out = gv.device_records(ctx, state["fmax"], gv.FACTOR_ACCUM_DTYPE)
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    if args.linearize_only:
        # profiling aid: S3-S7 alone on the last step's maps and factors
        lin_maps = gv.HandleArray(state["maps"])
        lin_fac = state["fac"]
        lin_pts = int(n_pts[lin_fac["source_cloud"]].sum())

        def step():  # noqa: F811
            gv.linearize_batch_accum(ctx, cloud_arr, lin_maps, lin_fac, poses,
                                     out=acc_out[:len(lin_fac)])
            return lin_pts, len(lin_fac)
        step()
        torch.cuda.synchronize()

    # ---- timed region
    clocks = ClockSampler(dev.index)
    if rank == 0:
        clocks.start()
        time.sleep(0.5)
    # per-kernel CUDA-event stage timing costs host time per launch: the
    # host-bound small configs (C1-C3) time their steps without it and take
    # the stage breakdown from a separate pass of the same steps afterwards
    stage_in_timed = args.config in ("C4", "C5")
    ctx.enable_timing(stage_in_timed)
    ctx.timing(reset=True)
    gv.launch_count(reset=True)
    for k_ in host_ms:
        host_ms[k_] = 0.0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    pts_total = 0
    fac_total = 0
    for _ in range(args.steps):
        p, f = step()
        pts_total += p
        fac_total += f
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = gv.launch_count(reset=True)
    clk = clocks.stop() if rank == 0 else None
    if not stage_in_timed:  # the stage breakdown: the same steps again, with event timing
        ctx.enable_timing(True)
        ctx.timing(reset=True)
        for k_ in host_ms:
            host_ms[k_] = 0.0
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
    tm = ctx.timing(reset=True)
    ctx.enable_timing(False)

    # max over ranks of the time; sum of the work
    if world > 1:
        t = torch.tensor([ms, pts_total, fac_total, launches], dtype=torch.float64, device=dev)
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms = float(tmax[0])
        pts_all, fac_all, launches_all = float(tsum[1]), float(tsum[2]), int(tsum[3])
    else:
        pts_all, fac_all, launches_all = float(pts_total), float(fac_total), launches
    ms_step = ms / args.steps
    value = pts_all / (ms / 1e3)

    # ---- SURVEY 8(d)'s per-call metric: ONE gvox_linearize_batch over the step's
    # selected factors, its single H2D (factor table + poses) and single D2H
    # (full records into pinned host memory) inside the interval, maps and clouds
    # resident (built once, amortised over GN iterations).  CUDA events on the
    # library's stream bracket the call (the host-side serialisation before the
    # H2D is inside the interval); median of >= 20 calls, max over ranks.
    per_call = None
    if not args.linearize_only and args.per_call_runs > 0:
        pc_fac = state["fac"]
        pc_maps = gv.HandleArray(state["maps"])
        pc_out = np.zeros(max(len(pc_fac), 1), gv.LINEAR_FACTOR_DTYPE)
        try:
            pc_out = torch.from_numpy(pc_out.view(np.uint8)).pin_memory().numpy().view(
                gv.LINEAR_FACTOR_DTYPE)
        except RuntimeError:
            pass
        pc_pts = int(n_pts[pc_fac["source_cloud"]].sum())
        gv.linearize_batch(ctx, cloud_arr, pc_maps, pc_fac, poses, out=pc_out[:len(pc_fac)])  # warm
        pc_ms = []
        for _ in range(args.per_call_runs):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            c0 = torch.cuda.Event(enable_timing=True)
            c1 = torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            gv.linearize_batch(ctx, cloud_arr, pc_maps, pc_fac, poses, out=pc_out[:len(pc_fac)])
            c1.record(stream)
            c1.synchronize()
            pc_ms.append(c0.elapsed_time(c1))
        med = statistics.median(pc_ms)
        pc_pf = float(pc_pts)
        pc_nf = float(len(pc_fac))
        if world > 1:
            t = torch.tensor([med, pc_pf, pc_nf], dtype=torch.float64, device=dev)
            tmax = t.clone()
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            tsum = t.clone()
            dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
            med, pc_pf, pc_nf = float(tmax[0]), float(tsum[1]), float(tsum[2])
        per_call = {"value": pc_pf / (med / 1e3), "unit": UNIT, "factors_per_s": pc_nf / (med / 1e3),
                    "ms_median": med, "ms_min": min(pc_ms), "ms_max": max(pc_ms),
                    "runs": len(pc_ms), "factors": int(pc_nf), "point_factors": int(pc_pf),
                    "h2d_bytes": int(pc_fac.nbytes + poses.nbytes),
                    "d2h_bytes": int(pc_out[:len(pc_fac)].nbytes),
                    "what": "one gvox_linearize_batch over the step's selected factors: one H2D "
                            "(factor table, poses), one fused launch, one D2H of full records "
                            "to pinned host memory (P:224); maps resident; median of the runs"}

    # ---- roofline of the dominant kernel (rank 0's launches)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else \
        "B200_PROFILING.md fallback 6.65 TB/s"
    fac = state["fac"]
    maps = state["maps"]
    lin_ms, lin_n = tm["linearize"]
    if args.linearize_only:
        log(f"[bench] linearize-only: {lin_ms / max(lin_n, 1):.3f} ms/launch, "
            f"{pts_all / (ms / 1e3):.4g} point-factors/s")
    # algorithmic bytes per launch: 48 B per point-factor (the 3 float4 source
    # planes) + compulsory map bytes (16 B slot + 48 B voxel record per voxel)
    # once per distinct target map in the launch.
    pf = int(n_pts[fac["source_cloud"]].sum())
    tmaps = np.unique(fac["target_map"])
    map_bytes = sum(64 * sum(maps[int(t)].num_voxels(l) for l in range(sc.levels)) for t in tmaps)
    alg_bytes = 48 * pf + map_bytes
    lin_avg_s = (lin_ms / max(lin_n, 1)) / 1e3
    achieved = alg_bytes / lin_avg_s / 1e9 if lin_n else None
    traffic = None
    inst_pf = None
    ncu = {}
    prof = os.path.join(ROOT, "profiles", "linearize_dram_bytes_per_pf.json")
    if os.path.exists(prof):
        try:
            ncu = json.load(open(prof))
            traffic = ncu["dram_bytes_per_point_factor"] * pf
            inst_pf = ncu.get("warp_instructions_per_point_factor")
        except (ValueError, KeyError):
            traffic = None
    # The kernel is bound by instruction issue (ncu: DRAM well below peak, no
    # pipe saturated, issue-active the highest utilisation), so the roofline
    # line is the ALU/issue ceiling: warp instructions per point-factor (the
    # committed full-size ncu capture) x point-factors / the live CUDA-event
    # launch time, against 4 schedulers x SMs x the SM clock sampled during the
    # timed region (one warp instruction per scheduler per cycle).
    # HBM is reported beside it two ways: measured DRAM bytes (ncu) and the
    # algorithmic-bytes model, each over the same live launch time.
    issue = None
    if inst_pf and lin_n and clk and clk.get("sm_mhz"):
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        peak_i = 4 * sms * clk["sm_mhz"] * 1e6
        ach_i = inst_pf * pf / lin_avg_s
        issue = {"achieved": ach_i / 1e9, "peak": peak_i / 1e9, "unit": "Gwarp-inst/s",
                 "frac": ach_i / peak_i, "warp_instructions_per_point_factor": inst_pf,
                 "peak_derivation": f"4 schedulers x {sms} SMs x {clk['sm_mhz']:.0f} MHz "
                                    "(1 warp-instruction / scheduler / cycle)"}
    hbm = {"peak": hbm_peak, "unit": "GB/s", "peak_source": peak_src,
           "measured_dram": {"achieved": traffic / lin_avg_s / 1e9 if (traffic and lin_n) else None,
                             "frac": (traffic / lin_avg_s / 1e9 / hbm_peak) if (traffic and lin_n) else None,
                             "bytes_per_point_factor": ncu.get("dram_bytes_per_point_factor"),
                             "source": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one "
                                       "full-size launch (profiles/linearize_dram_bytes_per_pf.json)"},
           "algorithmic": {"achieved": achieved, "frac": (achieved / hbm_peak) if achieved else None,
                           "bytes_per_launch": alg_bytes,
                           "model": "48 B per point-factor + 64 B per voxel of each distinct target"}}
    pipes = {k: ncu.get(k) for k in ("fma_pipe_pct", "alu_pipe_pct", "fp64_pipe_pct",
                                     "issue_active_pct", "dram_pct_of_peak", "occupancy_pct")
             if ncu.get(k) is not None}
    stages = {k: {"ms_per_step": v[0] / args.steps, "launches": v[1]} for k, v in tm.items()}
    # SURVEY §8(d) secondary rates (rank-local): per-row throughputs of the step
    rates = None
    if lin_n and tm["overlap"][1] and tm["build"][1]:
        try:
            inl = gv.records_to_numpy(acc_out[:len(fac)], gv.FACTOR_ACCUM_DTYPE)["inliers"]
            corr = int(inl.sum())
        except Exception:  # pragma: no cover
            corr = None
        tgt_pts = int(sum(n_pts[int(sc.map_clouds[t])] for t in my_targets))
        ovl_s = tm["overlap"][0] / tm["overlap"][1] / 1e3
        bld_s = tm["build"][0] / args.steps / 1e3
        rates = {"point_factors_per_s_linearize": pf / lin_avg_s,
                 "point_levels_per_s_linearize": pf * sc.levels / lin_avg_s,
                 "correspondences_per_s_linearize": (corr / lin_avg_s) if corr is not None else None,
                 "overlap_pairs_per_s": len(my_pairs) / ovl_s,
                 "overlap_points_per_s": float(src_n.sum()) / ovl_s,
                 "build_points_per_s": tgt_pts / bld_s}
    stages["host_wall_ms_per_step"] = {k: v / args.steps for k, v in host_ms.items()}
    dominant = max(tm, key=lambda k: tm[k][0])

    # ---- e2e through the public API with host buffers (rank-local, N GPUs)
    e2e = None
    if not args.no_e2e:
        # host inputs of this rank's shard (sources of its pairs and factors + its
        # targets), packed back to back in pinned memory
        need = set(int(c) for c in my_pairs[:, 0]) | set(int(sc.map_clouds[t]) for t in my_targets)
        if not select:
            need |= set(int(c) for c in fixed["source_cloud"])
        need = sorted(need)
        need_n = n_pts[need]
        loc_off = np.concatenate([[0], np.cumsum(need_n)]).astype(np.int64)
        tot_n = int(loc_off[-1])
        # the step's inputs: means and covariances, and normals only where the
        # step validates correspondences (C1-C3 odometry factors) --
        # the C4/C5 global factors never read them
        use_nrm = not select
        # one contiguous pinned block [means | covariances | normals]: the
        # upload is ONE copy (r02at, 8.7 MB: 179 us as one copy, 247 us as three)
        n_nrm = tot_n if use_nrm else 0
        host_flat = torch.empty(tot_n * 9 + n_nrm * 3, dtype=torch.float32).pin_memory()
        mu_h = host_flat[:3 * tot_n].view(tot_n, 3)
        cov_h = host_flat[3 * tot_n:9 * tot_n].view(tot_n, 6)
        nrm_h = host_flat[9 * tot_n:].view(n_nrm, 3)
        for j_, c_ in enumerate(need):
            a_, b_ = int(sc.offsets[c_]), int(sc.offsets[c_ + 1])
            mu_h[loc_off[j_]:loc_off[j_ + 1]] = torch.from_numpy(np.asarray(sc.mu[a_:b_]))
            cov_h[loc_off[j_]:loc_off[j_ + 1]] = torch.from_numpy(np.asarray(sc.cov[a_:b_]))
            if use_nrm:
                nrm_h[loc_off[j_]:loc_off[j_ + 1]] = torch.from_numpy(np.asarray(sc.nrm[a_:b_]))
        k_e2e = max(1, args.e2e_steps)
        # full records land in pinned host memory (a pageable D2H is staged at a
        # fraction of the PCIe rate)
        n_out = max(len(my_pairs), len(sc.factors), 1)
        pin_out = torch.empty(n_out * gv.LINEAR_FACTOR_DTYPE.itemsize, dtype=torch.uint8).pin_memory() \
            .numpy().view(gv.LINEAR_FACTOR_DTYPE)
        h2d = 0
        d2h = 0

        # Pipelined e2e (default, --e2e-mode pipelined): each step's inputs are copied from pinned host
        # memory into one of two device staging buffers on a copy stream, the
        # copy of step k + 1 overlapping the compute of step k (the way a
        # streaming deployment feeds the GPU); step k's clouds are then created
        # from the staged device arrays through the same public call.  Every
        # copy, including the first step's, is inside the timed region.
        # Default (serial): the copy inside each step, nothing overlapped.
        pipelined = args.e2e_mode == "pipelined"
        e2e_device_select = os.environ.get("GVOX_E2E_HOST_SELECT") is None
        # GVOX_E2E_ASYNC_READBACK=1: the result readback on a D2H stream,
        # double-buffered, overlapping the next step (r02ao, C5, 20 steps x 2:
        # 173.9 / 189.8 ms vs 177.7 / 177.4 synchronous -- no steadier gain)
        sync_readback = os.environ.get("GVOX_E2E_ASYNC_READBACK") is None
        early_upload = os.environ.get("GVOX_E2E_EARLY_UPLOAD") is not None
        if pipelined:
            stage_flat = [torch.empty(host_flat.shape, dtype=host_flat.dtype, device=dev) for _ in range(2)]
            stage = [(f_[:3 * tot_n].view(tot_n, 3), f_[3 * tot_n:9 * tot_n].view(tot_n, 6),
                      f_[9 * tot_n:].view(n_nrm, 3)) for f_ in stage_flat]
            cp_stream = torch.cuda.Stream(dev)
            pack_ev = [None, None]
            # the step's result (full records) expanded into one of two device
            # buffers and read back into pinned memory on a D2H stream, so the
            # readback of step k overlaps step k + 1 (the host does not wait
            # for it; the timed region ends after every copy has landed)
            if not sync_readback:
                rec_dev = [gv.device_records(ctx, n_out, gv.LINEAR_FACTOR_DTYPE) for _ in range(2)]
                rec_pin = [torch.empty((n_out, gv.LINEAR_FACTOR_DTYPE.itemsize), dtype=torch.uint8)
                           .pin_memory() for _ in range(2)]
            d2h_stream = torch.cuda.Stream(dev)
            d2h_ev = [None, None]

        def issue_h2d(k):
            """Upload step k's inputs into staging buffer k % 2 on the copy
            stream: three whole-array copies (the library's own small per-call
            inputs go through SM-driven copies, so they never queue behind
            this bulk upload on the copy engines); GVOX_E2E_CHUNK_MB > 0 uses
            pieces of that size from a helper thread, at most two in flight
            (the r01 scheme).  Returns (thread or None, [final event])."""
            b_ = k % 2
            done_ = []
            chunk_mb = float(os.environ.get("GVOX_E2E_CHUNK_MB", "0"))
            if chunk_mb <= 0:
                with torch.cuda.stream(cp_stream):
                    if pack_ev[b_] is not None:
                        cp_stream.wait_event(pack_ev[b_])
                    s_ = torch.cuda.Event(enable_timing=True)
                    s_.record(cp_stream)
                    stage_flat[b_].copy_(host_flat, non_blocking=True)  # one copy
                    e_ = torch.cuda.Event(enable_timing=True)
                    e_.record(cp_stream)
                    done_.append(e_)
                    done_.append(s_)
                return None, done_

            def run_():
                with torch.cuda.stream(cp_stream):
                    if pack_ev[b_] is not None:  # the buffer's previous step has packed it
                        cp_stream.wait_event(pack_ev[b_])
                    inflight_ = []
                    for dst_, src_ in zip(stage[b_], (mu_h, cov_h, nrm_h)):
                        rows_ = max(1, int(chunk_mb * (1 << 20)) // (src_.shape[1] * 4))
                        for r_ in range(0, src_.shape[0], rows_):
                            dst_[r_:r_ + rows_].copy_(src_[r_:r_ + rows_], non_blocking=True)
                            e_ = torch.cuda.Event()
                            e_.record(cp_stream)
                            inflight_.append(e_)
                            if len(inflight_) > 2:
                                e0_ = inflight_.pop(0)
                                while not e0_.query():  # (sleep releases the GIL)
                                    time.sleep(2e-4)
                    e_ = torch.cuda.Event()
                    e_.record(cp_stream)
                    done_.append(e_)

            th_ = threading.Thread(target=run_, daemon=True)
            th_.start()
            return th_, done_

        dbg_t = [time.perf_counter()]

        # GVOX_E2E_EVENTS=1: CUDA events at the phase boundaries (no syncs):
        # the GPU-side time from each boundary to the next, averaged over the
        # timed steps (idle gaps included), printed to stderr at the end
        ev_on = os.environ.get("GVOX_E2E_EVENTS") is not None
        ev_log = []

        def _dbg(what):
            if ev_on:
                e_ = torch.cuda.Event(enable_timing=True)
                e_.record(stream)
                ev_log.append((what, e_))
            if os.environ.get("GVOX_E2E_DEBUG"):
                t_ = time.perf_counter()
                log(f"[e2e] {what}: {1e3 * (t_ - dbg_t[0]):.1f} ms")
                dbg_t[0] = t_

        def e2e_step(k=0, ev_in=None, last=True):
            nonlocal h2d, d2h
            _dbg(f"step {k} start")
            ev_next = None
            if pipelined:
                if ev_in[0] is not None:
                    ev_in[0].join()  # every piece of step k's upload is enqueued
                stream.wait_event(ev_in[1][0])
                if os.environ.get("GVOX_E2E_DEBUG") and len(ev_in[1]) > 1:
                    ev_in[1][0].synchronize()
                    log(f"[e2e] upload of step {k}: {ev_in[1][1].elapsed_time(ev_in[1][0]):.1f} ms")
                # (C4/C5: step k + 1's upload is issued once this step's own
                # input blocks are on the device -- after the screened batch's
                # launch -- unless GVOX_E2E_EARLY_UPLOAD: the library's MB-sized
                # blocks are copied by SMs over PCIe and crawl behind a bulk
                # upload.  C1-C3: issued here, their blocks ride in launch
                # parameters)
                if not last and (early_upload or not (select and e2e_device_select)):
                    ev_next = issue_h2d(k + 1)
                b_ = k % 2
                cl_loc = gv.create_clouds(ctx, stage[b_][0], stage[b_][1],
                                          stage[b_][2] if use_nrm else None, loc_off)
                pe_ = torch.cuda.Event()
                pe_.record(stream)
                pack_ev[b_] = pe_
            else:
                cl_loc = gv.create_clouds(ctx, mu_h.numpy(), cov_h.numpy(),
                                          nrm_h.numpy() if use_nrm else None, loc_off)
            cl_all = [cl_loc[0]] * sc.num_clouds  # placeholders for clouds not used here
            for j_, c_ in enumerate(need):
                cl_all[c_] = cl_loc[j_]
            h2d_b = (48 if use_nrm else 36) * tot_n
            carr = gv.HandleArray(cl_all)
            _dbg("clouds")
            maps_e = gv.create_voxelmaps(ctx, [cl_all[int(sc.map_clouds[t])] for t in my_targets],
                                         sc.r0, sc.levels)
            marr = gv.HandleArray(maps_e)
            if select and e2e_device_select:
                # the screened batch through the public API with the decisions
                # kept on the device: gvox_overlap_select (device out) ->
                # gvox_linearize_batch_accum_select -> gvox_expand into pinned
                # host memory (full records: the step's result)
                _dbg("maps")
                gv.overlap_select(ctx, carr, marr, pairs_s, poses, sc.overlap_level, 1, 20,
                                  out=sel_d)
                ns = gv.linearize_batch_accum_select(ctx, carr, marr, all_fac, sel_d, poses,
                                                     acc_out, selected_host=sel_h)
                if pipelined and not last and not early_upload:
                    ev_next = issue_h2d(k + 1)
                _dbg("select + linearize")
                fe = all_fac[sel_h.view(bool)]
                cnt = sel_h
                if pipelined and not sync_readback:
                    b_ = k % 2
                    if d2h_ev[b_] is not None:  # this buffer's previous readback has landed
                        stream.wait_event(d2h_ev[b_])
                    gv.expand(ctx, fe, poses, acc_out[:ns], out=rec_dev[b_][:ns])
                    ex_ = torch.cuda.Event()
                    ex_.record(stream)
                    with torch.cuda.stream(d2h_stream):
                        d2h_stream.wait_event(ex_)
                        rec_pin[b_][:ns].copy_(rec_dev[b_][:ns], non_blocking=True)
                        dn_ = torch.cuda.Event()
                        dn_.record(d2h_stream)
                        d2h_ev[b_] = dn_
                    res = rec_pin[b_][:ns]
                else:
                    res = gv.expand(ctx, fe, poses, acc_out[:ns], out=pin_out[:ns])
                _dbg("expand")
            else:
                if select:
                    _dbg("maps")
                    cnt = gv.overlap_select(ctx, carr, marr, pairs_s, poses, sc.overlap_level, 1, 20)
                    _dbg("select")
                    fe = all_fac[cnt.view(bool)]
                else:
                    # (the counts stay on the device, as in the timed step: the
                    # factor list does not depend on them; the step's result
                    # read back is the linearization below)
                    gv.overlap(ctx, carr, marr, pairs_s, poses, sc.overlap_level, out=counts_d)
                    cnt = np.zeros(0, np.int32)
                    fe = fixed
                res = gv.linearize_batch(ctx, carr, marr, fe, poses, out=pin_out[:len(fe)])
                _dbg("linearize")
            h2d = h2d_b + poses.nbytes * 2 + pairs_s.nbytes + fe.nbytes
            d2h = cnt.nbytes + res.nbytes
            return int(n_pts[fe["source_cloud"]].sum()), ev_next

        def e2e_run(k_steps):
            ev_ = issue_h2d(0) if pipelined else None
            pts_ = 0
            for k_ in range(k_steps):
                p_, ev_ = e2e_step(k_, ev_, last=k_ == k_steps - 1)
                pts_ += p_
            return pts_

        e2e_run(1)  # warm-up
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        p_e2e = e2e_run(k_e2e)
        if pipelined:  # the interval ends after the last readback has landed
            for e_ in d2h_ev:
                if e_ is not None:
                    stream.wait_event(e_)
        a1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms_e2e = a0.elapsed_time(a1)
        if ev_on and ev_log:
            acc_ = {}
            for (w0, e0_), (w1, e1_) in zip(ev_log, ev_log[1:]):
                k_ = f"{w0.split(' ')[0]} -> {w1.split(' ')[0]}"
                acc_.setdefault(k_, []).append(e0_.elapsed_time(e1_))
            for k_, v_ in acc_.items():
                log(f"[e2e events] {k_}: {np.mean(v_):.3f} ms (n = {len(v_)})")
        if world > 1:
            t = torch.tensor([ms_e2e, p_e2e], dtype=torch.float64, device=dev)
            tm_ = t.clone()
            dist.all_reduce(tm_, op=dist.ReduceOp.MAX)
            ts_ = t.clone()
            dist.all_reduce(ts_, op=dist.ReduceOp.SUM)
            ms_e2e, p_e2e = float(tm_[0]), float(ts_[1])
        e2e = {"value": p_e2e / (ms_e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": k_e2e, "ms_per_step": ms_e2e / k_e2e,
               "mode": ("pipelined: step k+1's H2D (copy stream, double-buffered device staging) "
                        "overlaps step k's compute" +
                        ("" if sync_readback else ", step k's result read back on a D2H stream while "
                         "step k+1 runs") + "; every copy inside the timed region")
               if pipelined else "serial: each step's H2D inside the step"}

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        pts_o, dt_o, desc, cores = oracle_sample(sc, select, budget_s=args.cpu_seconds)
        # the same oracle on one thread (single-thread and all-core rates)
        pts_1, dt_1, desc_1, _ = oracle_sample(sc, select, budget_s=args.cpu_seconds / 3,
                                               threads=1)
        cpu = {"value": pts_o / dt_o, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": desc, "seconds": dt_o, "cpu_model": cpu_model(),
               "single_thread": {"value": pts_1 / dt_1, "unit": UNIT, "cores": 1,
                                 "sample": desc_1, "seconds": dt_1}}

    if rank == 0:
        n_levels_vox = {l: int(sum(m.num_voxels(l) for m in maps)) for l in range(sc.levels)}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded LiDAR-shaped submaps, synth/)",
            "config": {"workload": workload_label(args, sc), "submaps": sc.num_clouds,
                       "points": int(len(sc.mu)), "candidate_pairs": int(len(sc.pairs)),
                       "factors_per_step": fac_all / args.steps, "levels": sc.levels, "r0": sc.r0,
                       "overlap_level": sc.overlap_level, "point_order": args.order,
                       "parallelism": (f"factor-sharded x{world} (targets), one {dist.get_backend()} "
                                       "all_gather of the compact records" if world > 1 else
                                       "one GPU (no collective)"),
                       "shard_balance": balance if world > 1 else None,
                       "shard_bounds": bounds if world > 1 else None,
                       "l2": "inputs larger than L2 (clouds %.1f GB + voxel records %.1f GB + "
                             "index grids on rank 0)"
                             % (len(sc.mu) * 48 / 1e9,
                                sum(64 * v for v in n_levels_vox.values()) / 1e9),
                       "step": "S1 build all target maps + S2 overlap of all candidate pairs + "
                               "selection (20*count > N) + S3-S7 linearize selected factors"},
            "factors_per_s": fac_all / (ms / 1e3),
            "precision": "per-point fp32 algebra; fp64 transform, voxel keys, residual base "
                         "and cross-thread accumulation",
            "stages": stages,
            "rates": rates,
            "roofline": ({"kernel": "k_linearize", "bound": "alu",
                          "limiter": "instruction issue and memory latency at 25 % occupancy "
                                     "(128 registers); HBM and the FP32 pipe are below their peaks",
                          "achieved": issue["achieved"], "peak": issue["peak"], "unit": issue["unit"],
                          "frac": issue["frac"], "traffic": traffic,
                          "peak_derivation": issue["peak_derivation"],
                          "warp_instructions_per_point_factor": inst_pf,
                          "hbm": hbm, "ncu_pipes_pct": pipes,
                          "point_factors_per_launch": pf, "avg_launch_ms": lin_avg_s * 1e3,
                          "dominant_kernel_group": dominant}
                         if issue else
                         {"kernel": "k_linearize", "bound": "hbm", "achieved": achieved,
                          "peak": hbm_peak, "unit": "GB/s",
                          "frac": (achieved / hbm_peak) if achieved else None, "traffic": traffic,
                          "note": "no ncu instruction count or clock sample: algorithmic bytes only",
                          "point_factors_per_launch": pf, "avg_launch_ms": lin_avg_s * 1e3,
                          "dominant_kernel_group": dominant}),
            "per_call": per_call,
            "e2e": e2e,
            "gpu_launches": launches_all,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
