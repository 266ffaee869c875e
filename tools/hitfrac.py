import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth, sys
sys.path.insert(0, '.')
import paper_2407_10344_b200 as gv
sc = synth.make("C5", n_submaps=300)
ctx = gv.Context(0)
clouds = gv.create_clouds(ctx, sc.mu, sc.cov, sc.nrm, sc.offsets) if hasattr(gv, "create_clouds") else None
maps = gv.create_voxelmaps(ctx, clouds, sc.r0, sc.levels)
sel = gv.overlap_select(ctx, clouds, maps, sc.pairs, sc.poses, sc.overlap_level, 1, 20)
p = sc.pairs[sel.view(bool)]
f = np.array([[a[0], a[1], a[2], a[3], 0] for a in p], np.int64)
out = gv.linearize_batch(ctx, clouds, maps, f, sc.poses)
n = np.diff(sc.offsets)[f[:, 0]]
inl = out["inliers"][:, :3].astype(np.float64)
print("factors", len(f), "pairs", len(sc.pairs))
print("hit fraction per level", inl.sum(0) / n.sum())
print("no-hit fraction (1 - level2 hits)", 1 - inl[:, 2].sum() / n.sum())
cnt = gv.overlap(ctx, clouds, maps, sc.pairs, sc.poses, sc.overlap_level)
nn = np.diff(sc.offsets)[sc.pairs[:, 0]]
print("rejected pairs: mean level-1 hit frac", (cnt[~sel.view(bool)] / nn[~sel.view(bool)]).mean())
print("selected pairs: mean level-1 hit frac", (cnt[sel.view(bool)] / nn[sel.view(bool)]).mean())
cnt2 = gv.overlap(ctx, clouds, maps, sc.pairs, sc.poses, 2)
print("rejected pairs: mean level-2 hit frac", (cnt2[~sel.view(bool)] / nn[~sel.view(bool)]).mean())
