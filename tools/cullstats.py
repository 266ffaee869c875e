"""How much exact chunk culling could remove on the C5-shaped workload: for a
sample of overlap-selected factors, the fraction of 32-point chunks whose
transformed box meets no occupied coarsest-level cell, by allowed cell-range
size, and the fraction of no-hit points.  numpy; GPU only for the selection."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
import paper_2407_10344_b200 as gv

sc = synth.make("C5", n_submaps=300)
ctx = gv.Context(0)
clouds = gv.create_clouds(ctx, sc.mu, sc.cov, sc.nrm, sc.offsets)
maps = gv.create_voxelmaps(ctx, clouds, sc.r0, sc.levels)
sel = gv.overlap_select(ctx, clouds, maps, sc.pairs, sc.poses, sc.overlap_level, 1, 20).view(bool)
which = os.environ.get("CULL_PAIRS", "selected")
fac = sc.pairs[sel] if which == "selected" else sc.pairs[~sel]
rs = np.random.default_rng(0)
sample = fac[rs.choice(len(fac), 200, replace=False)]
print("pairs:", which)
L = sc.levels
rc = sc.r0 * 2 ** (L - 1)


def T(p):
    return np.asarray(p, np.float64).reshape(3, 4)


occ_cache = {}
res = {k: [0, 0] for k in (8, 27, 64, 10 ** 9)}
nohit_pts = tot_pts = 0
for s, t, pi, pj in sample:
    if t not in occ_cache:
        mu_t = sc.cloud(int(sc.map_clouds[t]))[0].astype(np.float64)
        occ_cache[t] = set(map(tuple, np.floor(mu_t / rc).astype(np.int64)))
    occ = occ_cache[t]
    Ti, Tj = T(sc.poses[pi]), T(sc.poses[pj])
    Ri, ti, Rj, tj = Ti[:, :3], Ti[:, 3], Tj[:, :3], Tj[:, 3]
    R = Rj.T @ Ri
    tt = Rj.T @ (ti - tj)
    mu = sc.cloud(int(s))[0].astype(np.float64)
    q = mu @ R.T + tt
    cells = np.floor(q / rc).astype(np.int64)
    hit = np.array([tuple(c) in occ for c in cells])
    nohit_pts += (~hit).sum()
    tot_pts += len(mu)
    n = len(mu)
    for c0 in range(0, n, 32):
        m = mu[c0:c0 + 32]
        lo, hi = m.min(0), m.max(0)
        ctr, h = (lo + hi) / 2, (hi - lo) / 2
        qc = R @ ctr + tt
        qh = np.abs(R) @ h + 1e-3
        clo = np.floor((qc - qh) / rc).astype(int)
        chi = np.floor((qc + qh) / rc).astype(int)
        ncell = np.prod(chi - clo + 1)
        empty = all(tuple((x, y, z)) not in occ for x in range(clo[0], chi[0] + 1)
                    for y in range(clo[1], chi[1] + 1) for z in range(clo[2], chi[2] + 1)) \
            if ncell <= 512 else False
        for k in res:
            res[k][1] += len(m)
            if empty and ncell <= k:
                res[k][0] += len(m)
print("no-hit point fraction", nohit_pts / tot_pts)
for k, (c, t) in res.items():
    print(f"max cells {k}: culled point fraction {c / t:.3f}")
