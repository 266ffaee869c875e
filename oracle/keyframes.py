"""Oracle of the keyframe mechanism.

TEST INFRASTRUCTURE ONLY (imported by tests/).  Plain Python written from the
paper, step by step:

  P:280  overlap rate o(i, j) = fraction of the points of P_i that fall within
         a voxel of P_j;  a new frame is inserted into the keyframe list if its
         overlap with the UNION of all keyframes is smaller than 90 %.
  P:282  1. remove keyframes that overlap the latest keyframe by less than 5 %;
  P:283  2. if more than N_odom keyframes exist, remove the keyframe that
            minimises s(i) = o(i, N_odom) * sum_{j in [1, N_odom-1] \\ {i}} (1 - o(i, j))
         (reading R25: the latest keyframe plays N_odom; j runs over
         the other non-latest keyframes that remain; ties -> the first one).
"""
from __future__ import annotations

import numpy as np

from . import oracle as _o


def keyframe_update(o, n_odom=20, min_overlap=0.05):
    """o: [K, K] overlap rates in list order, K-1 = the latest keyframe.
    Returns the list of removed positions."""
    K = len(o)
    latest = K - 1
    removed = set()
    for i in range(latest):                     # rule 1
        if o[i][latest] < min_overlap:
            removed.add(i)
    remaining = [i for i in range(K) if i not in removed]
    if len(remaining) > n_odom:                 # rule 2, one removal
        best, best_s = None, None
        for i in remaining:
            if i == latest:
                continue
            s = o[i][latest] * sum(1.0 - o[i][j] for j in remaining if j != i and j != latest)
            if best is None or s < best_s:
                best, best_s = i, s
        removed.add(best)
    return sorted(removed)


def run_keyframes(clouds, maps, poses, frames, level, n_odom=20, min_overlap=0.05):
    """Feed `frames` (indices into clouds / maps / poses) one by one through the
    insertion test and the removal rules.  Returns the keyframe list after each
    frame and the per-frame (inserted, removed) events."""
    kf = []
    events = []
    for f in frames:
        mu = clouds[f][0]
        n = len(mu)
        if kf:
            cnt = _o.overlap_union(mu, [maps[k] for k in kf], poses[f],
                                   np.stack([poses[k] for k in kf]), level)
            if not 10 * cnt < 9 * n:            # "smaller than 90 %", in integers
                events.append((False, []))
                continue
        ks = kf + [f]
        K = len(ks)
        o = np.zeros((K, K))
        for a in range(K):
            for b in range(K):
                na = len(clouds[ks[a]][0])
                c = _o.overlap(clouds[ks[a]][0], maps[ks[b]], poses[ks[a]], poses[ks[b]], level)
                o[a, b] = c / na if na else 0.0
        rm = keyframe_update(o, n_odom, min_overlap)
        events.append((True, [ks[a] for a in rm]))
        kf = [ks[a] for a in range(K) if a not in rm]
    return kf, events
