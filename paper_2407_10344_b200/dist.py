"""Multi-GPU plumbing for the batched linearization (one process per GPU,
torch.distributed over NCCL; gloo for the CPU tests of this host logic).

Factors are independent (Eqs. 2-8 per submap pair), so the batch shards by
TARGET map: each rank owns a contiguous range of target submaps, builds their
voxelmaps, screens their candidate pairs and linearizes the selected factors.
The only exchange is one all-gather of the fixed-size compact per-factor
records (gvox_factor_accum, 288 B) after linearization, so every rank (or the
host solver on rank 0) holds the whole linear system.
"""
from __future__ import annotations

import numpy as np


def shard_targets(n_points: np.ndarray, map_clouds: np.ndarray, pairs: np.ndarray,
                  world: int) -> list:
    """Contiguous target-map ranges [bounds[r], bounds[r+1]) balanced by the work
    each target attracts: its own points (map build) plus the source points of
    its candidate pairs (overlap + linearize).  pairs: int [P, >=2] with
    columns (source cloud, target map, ...)."""
    M = len(map_clouds)
    w = n_points[np.asarray(map_clouds)].astype(np.float64)
    if len(pairs):
        np.add.at(w, np.asarray(pairs)[:, 1], n_points[np.asarray(pairs)[:, 0]])
    cw = np.concatenate([[0.0], np.cumsum(w)])
    bounds = [0]
    for r in range(1, world):
        bounds.append(int(np.searchsorted(cw, cw[-1] * r / world)))
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
    """All-gather fixed-size records: `local` is a uint8 tensor [>= count, R]
    (the first `count` rows valid, padded to `fmax` rows); returns the
    concatenation of every rank's valid rows (rank order) and the counts.
    One all_gather_into_tensor of [world * fmax, R] bytes plus one tiny
    all_gather of the counts."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    R = local.shape[1]
    buf = local[:fmax] if local.shape[0] >= fmax else torch.cat(
        [local, local.new_zeros((fmax - local.shape[0], R))])
    cnt = torch.tensor([count], dtype=torch.int64, device=local.device)
    cnts = torch.empty(world, dtype=torch.int64, device=local.device)
    out = torch.empty((world * fmax, R), dtype=local.dtype, device=local.device)
    if local.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(cnts, cnt, group=group)
        dist.all_gather_into_tensor(out, buf.contiguous(), group=group)
    elif local.is_cuda:  # gloo with device tensors (plumbing tests): via the host
        o, c = gather_records(local.cpu(), count, fmax, group)
        return o.to(local.device), c
    else:  # gloo: list form
        cl = [torch.empty_like(cnt) for _ in range(world)]
        dist.all_gather(cl, cnt, group=group)
        cnts = torch.cat(cl)
        ol = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(ol, buf.contiguous(), group=group)
        out = torch.cat(ol)
    parts = [out[r * fmax: r * fmax + int(cnts[r])] for r in range(world)]
    return torch.cat(parts), [int(c) for c in cnts]


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
    [bounds[rank], bounds[rank + 1])).  Returns (delta, result, order)."""
    import paper_2407_10344_b200 as gv
    factors = np.asarray(factors)
    rows, loc = local_pairs(factors, bounds, rank)
    acc = gv.device_records(ctx, max(fmax, 1), gv.FACTOR_ACCUM_DTYPE)
    if len(loc):
        gv.linearize_batch_accum(ctx, clouds, maps_local, loc, poses, out=acc[:len(loc)])
    out, _ = gather_records(acc, len(loc), max(fmax, 1), group)
    order = shard_order(factors, bounds)
    delta, res, _, _ = gv.solve_global(ctx, factors[order], out.contiguous(), poses, fixed, **solve_kw)
    return delta, res, order
