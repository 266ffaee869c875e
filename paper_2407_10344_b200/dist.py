"""Multi-GPU plumbing for the batched linearization (one process per GPU,
torch.distributed over NCCL; gloo for the CPU tests of this host logic).

Factors are independent (Eqs. 2-8 per submap pair), so the batch shards by
TARGET map: each rank owns a contiguous range of target submaps, builds their
voxelmaps, screens their candidate pairs and linearizes the selected factors.
The only exchange is one all-gather of the fixed-size compact per-factor
records (gvox_factor_accum, 288 B; a header row carries each rank's count, so
it is a single collective) after linearization, so every rank (or the host
solver on rank 0) holds the whole linear system.  Shards
are balanced by the work each target attracts, using the previous step's
screening decisions when known (target_weights).
"""
from __future__ import annotations

import numpy as np


# Per-unit costs of the step's rows on one B200 at C5 (profiles/r02*_bench_c5.json
# stage times): S1 build ~8.3e-11 s per target point, S3-S7 linearize ~1.19e-11 s
# per selected point-factor, S2 screening ~6.5e-13 s per candidate source point
# (early exit makes it far cheaper than a lookup per point).  Only their RATIOS
# matter for balancing.
COST_BUILD = 7.0
COST_LINEARIZE = 1.0
COST_SCREEN = 0.055


def target_weights(n_points: np.ndarray, map_clouds: np.ndarray, pairs: np.ndarray,
                   selected: np.ndarray | None = None) -> np.ndarray:
    """Work each target map attracts, in linearize point-factor units: its own
    points (S1 build), the source points of its candidate pairs (S2 screening)
    and -- when the previous step's screening decisions `selected` (bool [P])
    are known -- the source points of its SELECTED pairs (S3-S7, the dominant
    row).  Without decisions every candidate counts as selected."""
    M = len(map_clouds)
    n_points = np.asarray(n_points)
    w = COST_BUILD * n_points[np.asarray(map_clouds)].astype(np.float64)
    if len(pairs):
        pairs = np.asarray(pairs)
        src = n_points[pairs[:, 0]].astype(np.float64)
        np.add.at(w, pairs[:, 1], COST_SCREEN * src)
        lin = src if selected is None else src * np.asarray(selected, bool)
        np.add.at(w, pairs[:, 1], COST_LINEARIZE * lin)
    assert len(w) == M
    return w


def shard_targets(n_points: np.ndarray, map_clouds: np.ndarray, pairs: np.ndarray,
                  world: int, weights: np.ndarray | None = None) -> list:
    """Contiguous target-map ranges [bounds[r], bounds[r+1]) balanced by the work
    each target attracts (`weights`, default target_weights without decisions).
    pairs: int [P, >=2] with columns (source cloud, target map, ...).  Contiguous
    ranges keep every factor of a target on one rank (its map built once, L2
    reuse of the map across those factors)."""
    M = len(map_clouds)
    w = target_weights(n_points, map_clouds, pairs) if weights is None else \
        np.asarray(weights, np.float64)
    assert len(w) == M
    cw = np.concatenate([[0.0], np.cumsum(w)])
    bounds = [0]
    for r in range(1, world):
        # the cut nearest to the ideal prefix (either side), not just the next one
        x = cw[-1] * r / world
        k = int(np.searchsorted(cw, x))
        if 0 < k <= M and abs(cw[k - 1] - x) < abs(cw[k] - x):
            k -= 1
        bounds.append(min(k, M))
    bounds.append(M)
    for r in range(world):  # monotone, within [0, M]
        bounds[r + 1] = max(bounds[r + 1], bounds[r])
    return bounds


def local_pairs(pairs: np.ndarray, bounds: list, rank: int):
    """(global row indices, local pairs with target re-indexed to the rank's
    map list) of the pairs whose target map this rank owns."""
    lo, hi = bounds[rank], bounds[rank + 1]
    pairs = np.asarray(pairs)
    rows = np.nonzero((pairs[:, 1] >= lo) & (pairs[:, 1] < hi))[0]
    loc = pairs[rows].copy()
    loc[:, 1] -= lo
    return rows, loc


def gather_records(local, count: int, fmax: int, group=None):
    """All-gather fixed-size records in ONE collective: `local` is a uint8
    tensor [>= count, R] whose first `count` rows are valid; every rank sends
    fmax + 1 rows -- a header row carrying its count (int64 in the first 8
    bytes), then its records padded to fmax -- with one all_gather_into_tensor
    (NCCL; gloo uses the list form).  Returns the concatenation of every rank's
    valid rows (rank order) and the counts.  count > fmax raises (the padded
    slot of a rank would spill into the next rank's)."""
    import torch
    import torch.distributed as dist
    if count > fmax or count > local.shape[0] or count < 0:
        raise ValueError(f"gather_records: count {count} exceeds fmax {fmax} or the "
                         f"{local.shape[0]} local rows")
    world = dist.get_world_size(group)
    R = local.shape[1]
    if R < 8:
        raise ValueError("gather_records: records narrower than the 8-byte count header")
    send = local.new_zeros((fmax + 1, R))
    if R % 8 == 0:  # device-side fill, no host copy
        send[0].view(torch.int64)[0].fill_(count)
    else:
        send[0, :8].copy_(torch.tensor([count], dtype=torch.int64).view(torch.uint8))
    if count:
        send[1:1 + count].copy_(local[:count])
    if local.is_cuda and dist.get_backend(group) == "nccl":
        out = torch.empty((world * (fmax + 1), R), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, send, group=group)
    elif local.is_cuda:  # gloo with device tensors (plumbing tests): via the host
        o, c = gather_records(local[:count].cpu(), count, fmax, group)
        return o.to(local.device), c
    else:  # gloo: list form
        ol = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(ol, send, group=group)
        out = torch.cat(ol)
    hdr = out.view(world, fmax + 1, R)[:, 0, :8].contiguous().cpu().numpy().view(np.int64).reshape(-1)
    cnts = [int(c) for c in hdr]
    parts = [out[r * (fmax + 1) + 1: r * (fmax + 1) + 1 + cnts[r]] for r in range(world)]
    return torch.cat(parts), cnts


def max_count(count: int, device=None, group=None) -> int:
    """fmax = the largest per-rank record count (one all_reduce MAX; setup, not
    per step)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(count)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())


def shard_order(factors: np.ndarray, bounds: list) -> np.ndarray:
    """Global factor rows in gathered (rank, then local) order."""
    return np.concatenate([local_pairs(factors, bounds, r)[0] for r in range(len(bounds) - 1)])


def global_step_sharded(ctx, clouds, maps_local, factors, bounds, rank: int, poses, fixed,
                        fmax: int, group=None, **solve_kw):
    """One Gauss-Newton step of the whole graph with the linearization sharded
    by target map (SURVEY §8(f) NEXT-4 on N GPUs): each rank linearizes its
    factors into compact records, ONE all-gather of the records (NCCL over
    NVLink), then every rank assembles and solves the same system
    (gvox_solve_global) in the same factor order, so all ranks hold bitwise
    the same step.  maps_local: the rank's target maps (targets
    [bounds[rank], bounds[rank + 1])).  fmax: the largest per-rank factor
    count (None: one all_reduce MAX).  Returns (delta, result, order)."""
    import paper_2407_10344_b200 as gv
    factors = np.asarray(factors)
    rows, loc = local_pairs(factors, bounds, rank)
    if fmax is None:
        fmax = max_count(len(loc), ctx.device, group)
    if len(loc) > fmax:
        raise ValueError(f"global_step_sharded: rank {rank} holds {len(loc)} factors > fmax {fmax}")
    acc = gv.device_records(ctx, max(fmax, 1), gv.FACTOR_ACCUM_DTYPE)
    if len(loc):
        gv.linearize_batch_accum(ctx, clouds, maps_local, loc, poses, out=acc[:len(loc)])
    out, _ = gather_records(acc, len(loc), max(fmax, 1), group)
    order = shard_order(factors, bounds)
    delta, res, _, _ = gv.solve_global(ctx, factors[order], out.contiguous(), poses, fixed, **solve_kw)
    return delta, res, order
