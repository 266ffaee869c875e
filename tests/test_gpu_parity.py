"""CUDA path (libgvox.so through the C ABI) vs the fp64 oracle, element by element.

Bars (BASELINE.json north_star): voxel keys, voxel counts, correspondences
(packed keys) and overlap counts bit-exact; H and b within 1e-4 relative
Frobenius error, e within 1e-5 (tests/parity.py).  Sizes span several tiles and
a ragged tail; edge cases: empty clouds, zero-hit factors, degenerate
covariances, validation, non-dyadic resolutions, out-of-range keys.
"""
import json
import os

import numpy as np
import pytest

import synth
from tests.parity import Margins, compare_factor
from tests.se3 import plane_cov, random_pose, rel_pose, right_perturb, to12, to44

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


@pytest.fixture(scope="module")
def ctx(gv):
    return gv.Context(0)


def rand_scene(rs, n, extent=20.0):
    """Plane-like Gaussian points on a few surfaces (like tests/test_oracle_linearize)."""
    normals = rs.normal(0, 1, (6, 3))
    normals /= np.linalg.norm(normals, axis=1, keepdims=True)
    pts, covs, nrms = [], [], []
    which = rs.integers(0, 6, n)
    for k in range(n):
        nv = normals[which[k]]
        t1 = np.cross(nv, [0.3, 0.5, 0.7]); t1 /= np.linalg.norm(t1)
        t2 = np.cross(nv, t1)
        p = nv * which[k] * 1.3 + t1 * rs.uniform(-extent, extent) + t2 * rs.uniform(-extent, extent)
        pts.append(p)
        covs.append(plane_cov(nv + rs.normal(0, 0.05, 3)))
        nrms.append(nv)
    return np.array(pts, np.float32), np.array(covs, np.float32), np.array(nrms, np.float32)


def transform_cloud(mu, cov, nrm, T12):
    """Express world-frame points in the frame of pose T (world <- frame)."""
    T = to44(T12)
    R, t = T[:3, :3], T[:3, 3]
    m = (mu.astype(float) - t) @ R
    C = np.zeros((len(cov), 3, 3))
    idx = [(0, 0, 0), (0, 1, 1), (0, 2, 2), (1, 1, 3), (1, 2, 4), (2, 2, 5)]
    for a, b, c in idx:
        C[:, a, b] = cov[:, c]
        C[:, b, a] = cov[:, c]
    C = np.einsum("ji,njk,kl->nil", R, C, R)
    c6 = np.stack([C[:, a, b] for a, b, _ in idx], 1)
    return m.astype(np.float32), c6.astype(np.float32), (nrm.astype(float) @ R).astype(np.float32)


# ---------------------------------------------------------------------- voxelmap
@pytest.mark.parametrize("r0,L,n,seed", [(0.25, 3, 20000, 0), (0.5, 3, 5000, 1), (0.3, 2, 7000, 2),
                                         (1.0, 1, 1000, 3), (0.125, 4, 3001, 4)])
def test_voxelmap_parity(gv, ctx, oracle, r0, L, n, seed):
    rs = np.random.default_rng(seed)
    mu, cov, nrm = rand_scene(rs, n)
    cl = gv.Cloud(ctx, mu, cov, nrm)
    m = gv.create_voxelmap(ctx, cl, r0, L)
    om = oracle.VoxelMap(mu, cov, r0, L)
    for l in range(L):
        keys, means, covs, counts = m.export(ctx, l)
        okeys, omeans, ocovs, ocounts = om.export(l)
        assert np.array_equal(keys, okeys), f"level {l}: keys differ"
        assert np.array_equal(counts.astype(np.int64), ocounts)
        r = r0 * 2 ** l
        np.testing.assert_allclose(means, omeans, rtol=0, atol=2e-7 * r + 1e-6 * 0)
        cmax = np.abs(cov).max()
        np.testing.assert_allclose(covs, ocovs, rtol=0, atol=2e-7 * cmax)


def test_voxelmap_batched_equals_single(gv, ctx):
    rs = np.random.default_rng(5)
    clouds = [gv.Cloud(ctx, *rand_scene(rs, n)) for n in (3000, 1, 0, 4500)]
    ms = gv.create_voxelmaps(ctx, clouds, 0.5, 3)
    for c, m in zip(clouds, ms):
        s = gv.create_voxelmap(ctx, c, 0.5, 3)
        for l in range(3):
            a, b = m.export(ctx, l), s.export(ctx, l)
            for x, y in zip(a, b):
                assert np.array_equal(x, y)


def test_voxelmap_batch_lifetime_and_recycling(gv, ctx):
    """A batch's maps go with ONE gvox_maps_destroy when the last of them does;
    a map closed explicitly before that is not destroyed twice; the record
    arenas and grids the batches release are recycled by the next builds of
    the same size, which still give identical maps."""
    import gc
    rs = np.random.default_rng(9)
    data = [rand_scene(rs, n) for n in (4000, 2500, 3000)]
    clouds = [gv.Cloud(ctx, *d) for d in data]
    ref = [[m.export(ctx, l) for l in range(3)] for m in gv.create_voxelmaps(ctx, clouds, 0.5, 3)]
    gc.collect()
    for rep in range(4):
        ms = gv.create_voxelmaps(ctx, clouds, 0.5, 3)
        assert [m.levels for m in ms] == [3, 3, 3]
        if rep % 2:
            ms[1].close()  # explicit close of one member, the rest with the batch
            ms[1].close()  # (idempotent)
        for i, m in enumerate(ms):
            if m.handle is None:
                continue
            got = [m.export(ctx, l) for l in range(3)]
            for a, b in zip(got, ref[i]):
                for x, y in zip(a, b):
                    assert np.array_equal(x, y)
        del ms
        gc.collect()


def test_voxelmap_golden_and_errors(gv, ctx, oracle):
    g = GOLDEN["two_points_voxel"]
    cl = gv.Cloud(ctx, np.array(g["mu"], np.float32), np.array(g["cov"], np.float32))
    m = gv.create_voxelmap(ctx, cl, g["r0"], 1)
    keys, means, covs, counts = m.export(ctx, 0)
    assert keys.tolist() == [oracle.pack_key(*g["voxel_key_xyz"])]
    np.testing.assert_allclose(means[0], g["mean"], atol=1e-7)
    np.testing.assert_allclose(covs[0], g["cov_mean"], atol=1e-6)
    assert counts.tolist() == [g["count"]]
    far = gv.Cloud(ctx, np.array([[3e6, 0, 0]], np.float32), np.ones((1, 6), np.float32))
    with pytest.raises(gv.GvoxError, match="GVOX_ERR_RANGE"):
        gv.create_voxelmap(ctx, far, 1.0, 1)
    with pytest.raises(gv.GvoxError, match="GVOX_ERR_INVALID"):
        gv.create_voxelmap(ctx, cl, 0.0, 1)
    with pytest.raises(gv.GvoxError, match="GVOX_ERR_INVALID"):
        gv.create_voxelmap(ctx, cl, 1.0, 9)
    with pytest.raises(gv.GvoxError, match="non-finite"):
        gv.Cloud(ctx, np.array([[np.nan, 0, 0]], np.float32), np.ones((1, 6), np.float32))


def test_lookup_parity(gv, ctx, oracle):
    rs = np.random.default_rng(6)
    mu, cov, nrm = rand_scene(rs, 4000, 10.0)
    for r0 in (0.5, 0.3):
        m = gv.create_voxelmap(ctx, gv.Cloud(ctx, mu, cov), r0, 3)
        om = oracle.VoxelMap(mu, cov, r0, 3)
        q = np.concatenate([mu[:500].astype(float) + rs.normal(0, 0.3, (500, 3)),
                            rs.uniform(-15, 15, (500, 3)),
                            np.round(mu[:200].astype(float) / r0) * r0])  # exact boundaries
        for l in range(3):
            got = m.lookup(ctx, l, q)
            want = np.array([om.lookup(l, p) for p in q])
            assert np.array_equal(got, want)


# ---------------------------------------------------------------------- overlap
def test_overlap_parity_random_poses(gv, ctx, oracle):
    rs = np.random.default_rng(7)
    mu, cov, nrm = rand_scene(rs, 6000, 15.0)
    srcs = [rand_scene(rs, n, 15.0)[0] for n in (5000, 2049, 1, 0, 4096)]
    clouds = [gv.Cloud(ctx, s, np.tile(cov[:1], (len(s), 1))) for s in srcs]
    maps = gv.create_voxelmaps(ctx, [gv.Cloud(ctx, mu, cov)], 0.5, 3)
    om = oracle.VoxelMap(mu, cov, 0.5, 3)
    poses = [to12(np.eye(4))] + [random_pose(rs, 0.05, 1.0) for _ in range(8)]
    pairs = [[s, 0, 1 + (s + k) % 8, 0] for s in range(len(srcs)) for k in range(3)]
    for level in range(3):
        got = gv.overlap(ctx, clouds, maps, pairs, poses, level)
        for p, g in zip(pairs, got):
            want = oracle.overlap(srcs[p[0]], om, poses[p[2]], poses[p[3]], level)
            assert int(g) == want


@pytest.mark.parametrize("num,den", [(1, 20), (0, 1), (1, 2), (19, 20), (1, 1), (3, 7)])
def test_overlap_select_matches_exact_decision(gv, ctx, oracle, num, den):
    """gvox_overlap_select stops early but must reproduce count * den > n * num."""
    rs = np.random.default_rng(17)
    mu, cov, nrm = rand_scene(rs, 8000, 12.0)
    srcs = [rand_scene(rs, n, 12.0)[0] for n in (9000, 2049, 1, 0, 4096, 777)]
    clouds = [gv.Cloud(ctx, s_, np.tile(cov[:1], (len(s_), 1))) for s_ in srcs]
    maps = gv.create_voxelmaps(ctx, [gv.Cloud(ctx, mu, cov)], 0.5, 3)
    om = oracle.VoxelMap(mu, cov, 0.5, 3)
    poses = [to12(np.eye(4))] + [random_pose(rs, 0.1 * k, 2.0 * k) for k in range(1, 9)]
    pairs = [[s_, 0, 1 + (s_ + k) % 8, 0] for s_ in range(len(srcs)) for k in range(4)]
    for level in (0, 1):
        got = gv.overlap_select(ctx, clouds, maps, pairs, poses, level, num, den)
        for p, g in zip(pairs, got):
            cnt = oracle.overlap(srcs[p[0]], om, poses[p[2]], poses[p[3]], level)
            assert int(g) == int(cnt * den > len(srcs[p[0]]) * num), (p, cnt, len(srcs[p[0]]))


def test_chunk_culling_exact(gv, ctx, oracle):
    """Spatially ordered sources sweeping across the map's edge: whole 32-point
    chunks are culled by their transformed bounding box (K2/K3).  The
    culled result must equal the oracle and, bit for bit, the unculled path
    (the correspondence dump disables culling), including points just inside
    the coarsest voxels that stick out of the map's own extent."""
    import torch
    rs = np.random.default_rng(23)
    # map: points on the slab x in [0, 10] (r0 = 0.5, L = 3: coarsest voxel 2 m)
    nm = 12000
    mu_m = np.stack([rs.uniform(0, 10, nm), rs.uniform(-5, 5, nm), rs.uniform(-1, 1, nm)], 1)
    mu_m[:5] = [10.0001, 0.5, 0.5]  # x max just past 10: level-2 voxel [10, 12) reaches 12.0001
    cov = np.tile(plane_cov(np.array([0.0, 0.0, 1.0]))[None], (nm, 1)).astype(np.float32)
    srcs = []
    for n, (a, b) in ((6000, (-20, 30)), (4000, (9.0, 12.5)), (3001, (-2.5, 1.0)), (700, (20, 40))):
        x = np.sort(rs.uniform(a, b, n))
        srcs.append(np.stack([x, rs.uniform(-6, 6, n), rs.uniform(-1.5, 1.5, n)], 1).astype(np.float32))
    # at the map box edge (x max + 2 m): x = 11.999 hits voxel [10, 12) of level 2
    srcs.append(np.array([[11.999, 0.1, 0.1]] * 40 + [[12.001, 0.1, 0.1]] * 40, np.float32))
    clouds = [gv.Cloud(ctx, s_, cov[:len(s_)] if len(s_) <= nm else np.tile(cov[:1], (len(s_), 1)))
              for s_ in srcs]
    m_cloud = gv.Cloud(ctx, mu_m.astype(np.float32), cov)
    maps = gv.create_voxelmaps(ctx, [m_cloud], 0.5, 3)
    om = oracle.VoxelMap(mu_m.astype(np.float32), cov, 0.5, 3)
    poses = [to12(np.eye(4))] + [random_pose(rs, 0.05, 0.5) for _ in range(4)]
    pairs = [[s_, 0, k % 5, 0] for s_ in range(len(srcs)) for k in range(3)]
    for level in range(3):
        got = gv.overlap(ctx, clouds, maps, pairs, poses, level)
        for p, g in zip(pairs, got):
            assert int(g) == oracle.overlap(srcs[p[0]], om, poses[p[2]], poses[p[3]], level), (p, level)
        sel = gv.overlap_select(ctx, clouds, maps, pairs, poses, level, 1, 4)
        n = np.array([len(srcs[p[0]]) for p in pairs])
        assert np.array_equal(sel.astype(bool), 4 * got.astype(np.int64) > n)
    fac = np.array([[p[0], 0, p[2], 0, 0] for p in pairs], np.int64)
    out = gv.linearize_batch(ctx, clouds, maps, fac, poses)
    corr = torch.empty(gv.corr_dump_size(clouds, maps, fac), dtype=torch.int64, device=ctx.device)
    nocull = gv.linearize_batch(ctx, clouds, maps, fac, poses, corr_dump=corr)
    assert out.tobytes() == nocull.tobytes()
    assert list(out["inliers"][-3, :3]) == [0, 0, 40]  # identity pose: level 2 only
    for k, f in enumerate(fac):
        ref = oracle.linearize(srcs[f[0]], cov[:len(srcs[f[0]])], None, om, poses[f[2]], poses[f[3]])
        compare_factor(out[k], ref, 3, what=f"cull factor {k}")


def test_overlap_c2(gv, ctx, oracle):
    sc = synth.make("C2")
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    for level in range(sc.levels):
        got = gv.overlap(ctx, clouds, maps, sc.pairs, sc.poses, level)
        for p, g in zip(sc.pairs, got):
            om = oracle.VoxelMap(*sc.cloud(int(sc.map_clouds[p[1]]))[:2], sc.r0, sc.levels)
            want = oracle.overlap(sc.cloud(int(p[0]))[0], om, sc.poses[p[2]], sc.poses[p[3]], level)
            assert int(g) == want
        # cross-kernel identity: overlap count at level l = linearize inliers[l] (no validation)
    f = sc.factors.copy()
    f[:, 4] = 0
    out = gv.linearize_batch(ctx, clouds, maps, f, sc.poses)
    for level in range(sc.levels):
        got = gv.overlap(ctx, clouds, maps, sc.pairs, sc.poses, level)
        assert np.array_equal(got, out["inliers"][:, level])


# ---------------------------------------------------------------------- linearize
def _scene_parity(gv, ctx, oracle, sc, check_corr=True, margins=None):
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    import torch
    corr = None
    if check_corr:
        corr = torch.empty(gv.corr_dump_size(clouds, maps, sc.factors), dtype=torch.int64,
                           device=ctx.device)
    out = gv.linearize_batch(ctx, clouds, maps, sc.factors, sc.poses, corr_dump=corr)
    corr_h = corr.cpu().numpy() if check_corr else None
    omaps = {}
    off = 0
    mg = margins if margins is not None else Margins(sc.name)
    for k, f in enumerate(sc.factors):
        t = int(f[1])
        if t not in omaps:
            omaps[t] = oracle.VoxelMap(*sc.cloud(int(sc.map_clouds[t]))[:2], sc.r0, sc.levels)
        mu, cov, nrm = sc.cloud(int(f[0]))
        ref = oracle.linearize(mu, cov, nrm, omaps[t], sc.poses[f[2]], sc.poses[f[3]],
                               validate=bool(f[4] & 1), return_corr=check_corr)
        mg.add_ints("inliers", sc.levels, int((out[k]["inliers"][:sc.levels] != ref["inliers"]).sum()))
        mg.add_factor(compare_factor(out[k], ref, sc.levels, what=f"{sc.name} factor {k}"))
        if check_corr:
            n = len(mu) * sc.levels
            bad = int((corr_h[off:off + n] != ref["corr"].reshape(-1)).sum())
            mg.add_ints("correspondences", n, bad)
            assert bad == 0, f"factor {k} corr: {bad} mismatches"
            off += n
    return out, mg.worst, mg


def test_linearize_c1(gv, ctx, oracle):
    _scene_parity(gv, ctx, oracle, synth.make("C1"))[2].save("test_linearize_c1")


def test_linearize_c2_validation(gv, ctx, oracle):
    out, worst, mg = _scene_parity(gv, ctx, oracle, synth.make("C2"))
    assert out["inliers"][:, :3].min() > 0
    mg.save("test_linearize_c2_validation")


def test_linearize_c3_subset(gv, ctx, oracle):
    sc = synth.make("C3")
    sc.factors = sc.factors[::7].copy()  # 43 of 300 factors, all 50 clouds uploaded
    _scene_parity(gv, ctx, oracle, sc)[2].save("test_linearize_c3_subset")


def test_linearize_random_factors_nondyadic(gv, ctx, oracle):
    rs = np.random.default_rng(11)
    mu_w, cov_w, n_w = rand_scene(rs, 9000, 12.0)
    Ts = [random_pose(rs, 0.4, 4.0) for _ in range(5)]
    clouds = [transform_cloud(mu_w[k * 1500:(k + 1) * 1500 + 777], cov_w[k * 1500:(k + 1) * 1500 + 777],
                              n_w[k * 1500:(k + 1) * 1500 + 777], Ts[k]) for k in range(5)]
    poses = np.stack([right_perturb(T, rs.normal(0, 0.01, 6)) for T in Ts])
    mg = Margins("random non-dyadic (r0 0.3/0.7/0.25, L 3/1/5)")
    for r0, L in ((0.3, 3), (0.7, 1), (0.25, 5)):
        sc = synth.Scene("rand", np.concatenate([c[0] for c in clouds]),
                         np.concatenate([c[1] for c in clouds]), np.concatenate([c[2] for c in clouds]),
                         np.concatenate([[0], np.cumsum([len(c[0]) for c in clouds])]).astype(np.int64),
                         np.arange(5, dtype=np.int64), r0, L,
                         np.array([[i, j, i, j, (i + j) % 2] for i in range(5) for j in range(5) if i != j],
                                  np.int64), poses, poses, np.zeros((0, 4), np.int64), 0)
        _scene_parity(gv, ctx, oracle, sc, margins=mg)
    mg.save("test_linearize_random_factors_nondyadic")


def test_linearize_zero_at_ground_truth_lattice(gv, ctx):
    # dyadic lattice, 90-degree rotations: every fp op exact on both paths -> e = b = 0 exactly
    g = np.stack(np.meshgrid(np.arange(-2, 3), np.arange(-2, 3), np.arange(0, 2), indexing="ij"), -1).reshape(-1, 3)
    src = (g * 8.0 + np.array([1.5, 2.25, 3.125])).astype(np.float32)
    Rz = np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1.0]])
    Rx = np.array([[1, 0, 0], [0, 0, -1], [0, 1, 0.0]])
    Ti = np.eye(4); Ti[:3, :3] = Rz; Ti[:3, 3] = [16.0, -8.0, 0.0]
    Tj = np.eye(4); Tj[:3, :3] = Rx; Tj[:3, 3] = [-24.0, 8.0, 32.0]
    Tij = np.linalg.inv(Tj) @ Ti
    tgt = (src.astype(float) @ Tij[:3, :3].T + Tij[:3, 3]).astype(np.float32)
    cov = np.tile(np.array(plane_cov([0.3, 0.4, 0.866]), np.float32), (len(src), 1))
    cs, ct = gv.Cloud(ctx, src, cov), gv.Cloud(ctx, tgt, cov)
    m = gv.create_voxelmap(ctx, ct, 1.0, 3)
    out = gv.linearize_batch(ctx, [cs], [m], [[0, 0, 0, 1, 0]], np.stack([to12(Ti), to12(Tj)]))
    assert out["inliers"][0][:3].tolist() == [len(src)] * 3
    assert out["error"][0] == 0.0
    assert np.all(out["b_i"][0] == 0.0) and np.all(out["b_j"][0] == 0.0)


@pytest.mark.parametrize("name", ["d2d_unit", "d2d_rotated"])
def test_linearize_golden(gv, ctx, name):
    g = GOLDEN[name]
    ct = gv.Cloud(ctx, np.array(g["target_mu"], np.float32), np.array(g["target_cov"], np.float32))
    cs = gv.Cloud(ctx, np.array(g["source_mu"], np.float32), np.array(g["source_cov"], np.float32))
    m = gv.create_voxelmap(ctx, ct, g["r0"], g["levels"])
    out = gv.linearize_batch(ctx, [cs], [m], [[0, 0, 0, 1, 0]], np.stack([g["T_i"], g["T_j"]]))
    assert out["error"][0] == pytest.approx(g["e"], rel=1e-6)


def test_visibility_golden(gv, ctx):
    g = GOLDEN["visibility_wall"]
    mu = np.array([g["point"]], np.float32)
    unit = np.array([[1, 0, 0, 1, 0, 1]], np.float32)
    cs = gv.Cloud(ctx, mu, unit, np.array([g["normal"]], np.float32))
    for x, inv in zip(g["viewer_x"], g["invisible"]):
        m = gv.create_voxelmap(ctx, gv.Cloud(ctx, mu - np.array([[x, 0, 0]], np.float32), unit), 1.0, 1)
        poses = np.stack([np.eye(4)[:3].reshape(-1), np.array([1, 0, 0, x, 0, 1, 0, 0, 0, 0, 1, 0.0])])
        out = gv.linearize_batch(ctx, [cs], [m], [[0, 0, 0, 1, gv.F_VALIDATE_SURFACE]], poses)
        assert int(out["num_invisible"][0]) == inv
        assert int(out["inliers"][0][0]) == 1 - inv


def test_edge_cases(gv, ctx, oracle):
    rs = np.random.default_rng(12)
    mu, cov, nrm = rand_scene(rs, 3000, 8.0)
    full = gv.Cloud(ctx, mu, cov, nrm)
    empty = gv.Cloud(ctx, np.zeros((0, 3), np.float32), np.zeros((0, 6), np.float32))
    m = gv.create_voxelmap(ctx, full, 0.5, 3)
    m_empty = gv.create_voxelmap(ctx, empty, 0.5, 3)
    I = to12(np.eye(4))
    far = to44(I); far[0, 3] = 1e4
    poses = np.stack([I, to12(far)])
    f = [[1, 0, 0, 0, 0],   # empty source
         [0, 1, 0, 0, 0],   # empty target map
         [0, 0, 1, 0, 0],   # no overlap (far away)
         [0, 0, 0, 0, 0]]   # self
    out = gv.linearize_batch(ctx, [full, empty], [m, m_empty], f, poses)
    for k in range(3):
        assert out["error"][k] == 0 and np.all(out["H_jj"][k] == 0) and out["inliers"][k].sum() == 0
    ref = oracle.linearize(mu, cov, None, oracle.VoxelMap(mu, cov, 0.5, 3), I, I)
    compare_factor(out[3], ref, 3)
    # degenerate (exactly zero) covariances: skipped and counted (Q16)
    z = np.zeros((1, 6), np.float32)
    cz = gv.Cloud(ctx, np.array([[0.2, 0.5, 0.5]], np.float32), z)
    mz = gv.create_voxelmap(ctx, gv.Cloud(ctx, np.array([[0.5, 0.5, 0.5]], np.float32), z), 1.0, 1)
    out = gv.linearize_batch(ctx, [cz], [mz], [[0, 0, 0, 0, 0]], np.stack([I]))
    assert int(out["num_degenerate"][0]) == 1 and out["inliers"][0][0] == 0 and out["error"][0] == 0
    # argument errors name the factor
    with pytest.raises(gv.GvoxError, match="factor 1: pose_j 7 missing"):
        gv.linearize_batch(ctx, [full], [m], [[0, 0, 0, 0, 0], [0, 0, 0, 7, 0]], np.stack([I]))
    with pytest.raises(gv.GvoxError, match="factor 0: target_map 3"):
        gv.linearize_batch(ctx, [full], [m], [[0, 3, 0, 0, 0]], np.stack([I]))
    bad = np.stack([I]).copy(); bad[0, 3] = np.inf
    with pytest.raises(gv.GvoxError, match="not finite"):
        gv.linearize_batch(ctx, [full], [m], [[0, 0, 0, 0, 0]], bad)


def test_batch_equals_serial_and_determinism(gv, ctx):
    sc = synth.make("C2")
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    a = gv.linearize_batch(ctx, clouds, maps, sc.factors, sc.poses)
    b = gv.linearize_batch(ctx, clouds, maps, sc.factors, sc.poses)
    assert a.tobytes() == b.tobytes(), "repeated runs must be bitwise identical"
    # a factor's tiling depends on the factor alone: batch == serial bit for bit
    for k in range(len(sc.factors)):
        s = gv.linearize_batch(ctx, clouds, maps, sc.factors[k:k + 1], sc.poses)
        assert s[0].tobytes() == a[k].tobytes(), f"factor {k}"
    # N identical factors -> N identical outputs
    rep = np.repeat(sc.factors[:1], 5, axis=0)
    r = gv.linearize_batch(ctx, clouds, maps, rep, sc.poses)
    assert all(r[k].tobytes() == r[0].tobytes() for k in range(5))


@pytest.fixture(scope="module")
def dense_scene():
    # submaps (C4 recipe, small): every level gets a dense index grid
    return synth.global_scene(n_submaps=8, n_points=30000, half_blocks=2, factor_dist=40.0,
                              cand_dist=60.0)


@pytest.mark.parametrize("which", ["C2-hash", "C4-dense"])
@pytest.mark.parametrize("flags", [0, 1])
def test_fast_kernel_equals_generic(gv, ctx, monkeypatch, flags, which, request):
    """The specialised kernel (3 dyadic levels, no dump; dense-grid or hash
    levels; its VALID variant with the P:197 visibility test) performs the same
    arithmetic in the same order as the generic one."""
    sc = synth.make("C2") if which == "C2-hash" else request.getfixturevalue("dense_scene")
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    if which == "C2-hash":  # every level a hash table (zero dense-grid budget)
        monkeypatch.setenv("GVOX_DENSE_BUDGET_MB", "0")
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    monkeypatch.delenv("GVOX_DENSE_BUDGET_MB", raising=False)
    f = sc.factors.copy()
    f[:, 4] = flags
    fast = gv.linearize_batch(ctx, clouds, maps, f, sc.poses)
    monkeypatch.setenv("GVOX_LIN_GENERIC", "1")
    generic = gv.linearize_batch(ctx, clouds, maps, f, sc.poses)
    assert fast.tobytes() == generic.tobytes()
    assert fast["inliers"].sum() > 0
    assert (fast["num_invisible"].sum() > 0) == bool(flags)


def test_compact_expand_equals_full(gv, ctx):
    import torch
    sc = synth.make("C2")
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    full = gv.linearize_batch(ctx, clouds, maps, sc.factors, sc.poses)
    acc = gv.device_records(ctx, len(sc.factors), gv.FACTOR_ACCUM_DTYPE)
    gv.linearize_batch_accum(ctx, clouds, maps, sc.factors, sc.poses, out=acc)
    exp = gv.expand(ctx, sc.factors, sc.poses, acc)
    assert exp.tobytes() == full.tobytes()
    dev = gv.device_records(ctx, len(sc.factors), gv.LINEAR_FACTOR_DTYPE)
    gv.linearize_batch(ctx, clouds, maps, sc.factors, sc.poses, out=dev)
    torch.cuda.synchronize()
    assert gv.records_to_numpy(dev).tobytes() == full.tobytes()


def test_error_only_flag(gv, ctx):
    sc = synth.make("C2")
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    full = gv.linearize_batch(ctx, clouds, maps, sc.factors, sc.poses)
    f = sc.factors.copy()
    f[:, 4] |= gv.F_ERROR_ONLY
    eo = gv.linearize_batch(ctx, clouds, maps, f, sc.poses)
    assert np.array_equal(eo["error"], full["error"]) or np.allclose(eo["error"], full["error"], rtol=1e-12)
    assert np.all(eo["H_jj"] == 0) and np.array_equal(eo["inliers"], full["inliers"])


# ------------------------------------------------------------ full-size samples
def test_full_size_submaps_sampled(gv, ctx, oracle):
    """Per-factor sizes of C5 (100k-point submaps, r = 0.5/1/2 m) in the bench's
    launch configuration (one batch over all factors, validation off); a sample
    of factors and pairs is recomputed by the oracle."""
    sc = synth.make("C5", n_submaps=48, half_blocks=4)
    assert sc.cloud_size(0) == 100000
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, clouds, sc.r0, sc.levels)
    out = gv.linearize_batch(ctx, clouds, maps, sc.factors, sc.poses)
    cnt = gv.overlap(ctx, clouds, maps, sc.pairs, sc.poses, sc.overlap_level)
    rs = np.random.default_rng(0)
    omaps = {}
    for k in rs.choice(len(sc.factors), 6, replace=False):
        f = sc.factors[k]
        t = int(f[1])
        omaps.setdefault(t, oracle.VoxelMap(*sc.cloud(t)[:2], sc.r0, sc.levels))
        mu, cov, nrm = sc.cloud(int(f[0]))
        ref = oracle.linearize(mu, cov, nrm, omaps[t], sc.poses[f[2]], sc.poses[f[3]])
        compare_factor(out[k], ref, sc.levels, what=f"C5-size factor {k}")
    sel = gv.overlap_select(ctx, clouds, maps, sc.pairs, sc.poses, sc.overlap_level, 1, 20)
    n = np.diff(sc.offsets)
    assert np.array_equal(sel.astype(bool), 20 * cnt.astype(np.int64) > n[sc.pairs[:, 0]])
    for k in rs.choice(len(sc.pairs), 6, replace=False):
        p = sc.pairs[k]
        t = int(p[1])
        omaps.setdefault(t, oracle.VoxelMap(*sc.cloud(t)[:2], sc.r0, sc.levels))
        want = oracle.overlap(sc.cloud(int(p[0]))[0], omaps[t], sc.poses[p[2]], sc.poses[p[3]],
                              sc.overlap_level)
        assert int(cnt[k]) == want
        assert int(sel[k]) == int(20 * want > n[int(p[0])])
    # one sampled map, exported and compared bit-exactly on keys/counts
    t = int(sc.factors[0][1])
    omaps.setdefault(t, oracle.VoxelMap(*sc.cloud(t)[:2], sc.r0, sc.levels))
    for l in range(sc.levels):
        keys, means, covs, counts = maps[t].export(ctx, l)
        okeys, omeans, ocovs, ocounts = omaps[t].export(l)
        assert np.array_equal(keys, okeys) and np.array_equal(counts.astype(np.int64), ocounts)


@pytest.mark.slow
@pytest.mark.parametrize("config", ["C4", "C5"])
def test_full_bench_configuration_sampled(gv, ctx, oracle, config):
    """The bench's own workload and launch configuration at full size (C5:
    2000 submaps x 100k points, ~2e5 candidate pairs; C4: 500 x 50k), one
    gvox_overlap_select over every candidate, one gvox_linearize_batch_accum
    over the ~1e5 selected factors (FAST all-dense kernel), the device-compacted
    select path bitwise equal to it, and sampled outputs the oracle computes one
    by one: 32 target submaps (the 16 farthest from the world origin + 16
    random), >= 256 screening decisions against the oracle's exact counts,
    64 factors (records expanded from the big batch) against the oracle's
    factors, and the same 64 factors' correspondences (packed voxel keys of
    every point at every level) dumped at these coordinates and
    compared bit for bit; the FAST kernel's records for them equal the generic
    (dumping) kernel's bitwise."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    sc = synth.make(config)
    clouds = gv.create_clouds(ctx, torch.from_numpy(sc.mu).cuda(), torch.from_numpy(sc.cov).cuda(),
                              torch.from_numpy(sc.nrm).cuda(), sc.offsets)
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    sel = gv.overlap_select(ctx, clouds, maps, sc.pairs, sc.poses, sc.overlap_level, 1, 20)
    cnt = gv.overlap(ctx, clouds, maps, sc.pairs, sc.poses, sc.overlap_level)
    n = np.diff(sc.offsets)
    assert np.array_equal(sel.astype(bool), 20 * cnt.astype(np.int64) > n[sc.pairs[:, 0]])
    fac = np.zeros(len(sc.pairs), gv.FACTOR_DTYPE)
    for i, name in enumerate(("source_cloud", "target_map", "pose_i", "pose_j")):
        fac[name] = sc.pairs[:, i]
    cand = fac
    fac = fac[sel.view(bool)]
    assert len(fac) > (100000 if config == "C5" else 10000)
    acc = gv.device_records(ctx, len(fac), gv.FACTOR_ACCUM_DTYPE)
    gv.linearize_batch_accum(ctx, clouds, maps, fac, sc.poses, out=acc)
    # the bench's call sequence: device decisions -> device-compacted batch,
    # bitwise the two-call path's records
    dsel = torch.empty(len(sc.pairs), dtype=torch.uint8, device=ctx.device)
    gv.overlap_select(ctx, clouds, maps, sc.pairs, sc.poses, sc.overlap_level, 1, 20, out=dsel)
    acc2 = gv.device_records(ctx, len(cand), gv.FACTOR_ACCUM_DTYPE)
    sel_h = np.zeros(len(cand), np.uint8)
    ns = gv.linearize_batch_accum_select(ctx, clouds, maps, cand, dsel, sc.poses, acc2,
                                         selected_host=sel_h)
    assert ns == len(fac) and np.array_equal(sel_h, sel)
    assert torch.equal(acc2[:ns], acc)
    del acc2

    mg = Margins(f"{config} full size (sampled)")
    rs = np.random.default_rng(7)
    pos = sc.poses.reshape(-1, 3, 4)[:, :, 3]
    tsel = np.unique(fac["target_map"])
    far = tsel[np.argsort(-np.linalg.norm(pos[sc.map_clouds[tsel]], axis=1), kind="stable")[:16]]
    rest = rs.choice(np.setdiff1d(tsel, far), 16, replace=False)
    targets = [int(t) for t in np.concatenate([far, rest])]
    with ThreadPoolExecutor(16) as ex:
        ol = list(ex.map(lambda t: oracle.VoxelMap(*sc.cloud(int(sc.map_clouds[t]))[:2], sc.r0,
                                                   sc.levels), targets))
    local = {t: k for k, t in enumerate(targets)}

    # >= 256 screening decisions: 8 candidate pairs per sampled target, half
    # selected where possible
    dk = []
    for t in targets:
        idx = np.nonzero(sc.pairs[:, 1] == t)[0]
        on, off = idx[sel[idx] == 1], idx[sel[idx] == 0]
        k_off = min(4, len(off))
        dk += rs.choice(on, min(8 - k_off, len(on)), replace=False).tolist()
        dk += rs.choice(off, k_off, replace=False).tolist() if k_off else []
    dk = np.array(sorted(dk))
    assert len(dk) >= 256
    lp = sc.pairs[dk].copy()
    lp[:, 1] = [local[int(t)] for t in lp[:, 1]]
    want = oracle.overlap_batch([sc.cloud(c)[0] for c in range(sc.num_clouds)], ol, lp, sc.poses,
                                sc.overlap_level, num_threads=16)
    assert np.array_equal(cnt[dk].astype(np.int64), want)
    wsel = (20 * want > n[sc.pairs[dk, 0]]).astype(np.uint8)
    mg.add_ints("overlap counts", len(dk), int((cnt[dk] != want).sum()))
    mg.add_ints("screening decisions", len(dk), int((sel[dk] != wsel).sum()))
    assert np.array_equal(sel[dk], wsel)

    # 64 factors: two selected factors per sampled target
    pick = []
    for t in targets:
        idx = np.nonzero(fac["target_map"] == t)[0]
        pick += rs.choice(idx, min(2, len(idx)), replace=False).tolist()
    pick = np.array(sorted(pick))
    assert len(pick) >= 64
    sub = gv.device_records(ctx, len(pick), gv.FACTOR_ACCUM_DTYPE)
    sub.copy_(acc[torch.from_numpy(pick).cuda()])
    full = gv.records_to_numpy(gv.expand(ctx, fac[pick], sc.poses, sub,
                                         out=gv.device_records(ctx, len(pick), gv.LINEAR_FACTOR_DTYPE)))
    fsub = fac[pick]
    corr = torch.empty(gv.corr_dump_size(clouds, maps, fsub), dtype=torch.int64, device=ctx.device)
    dumped = gv.linearize_batch(ctx, clouds, maps, fsub, sc.poses, corr_dump=corr)   # generic kernel
    fast = gv.linearize_batch(ctx, clouds, maps, fsub, sc.poses)                     # FAST kernel
    assert dumped.tobytes() == fast.tobytes()
    assert fast.tobytes() == full.tobytes()      # a factor's result is independent of its batch
    corr_h = corr.cpu().numpy()

    def ref_of(f):
        mu, cov, _ = sc.cloud(int(f["source_cloud"]))
        return oracle.linearize(mu, cov, None, ol[local[int(f["target_map"])]], sc.poses[f["pose_i"]],
                                sc.poses[f["pose_j"]], return_corr=True)

    with ThreadPoolExecutor(16) as ex:
        refs = list(ex.map(ref_of, fsub))
    off = 0
    for j, (f, ref) in enumerate(zip(fsub, refs)):
        mg.add_ints("inliers", sc.levels, int((full[j]["inliers"][:sc.levels] != ref["inliers"]).sum()))
        mg.add_factor(compare_factor(full[j], ref, sc.levels, what=f"{config} factor {pick[j]}"))
        m = n[int(f["source_cloud"])] * sc.levels
        bad = int((corr_h[off:off + m] != ref["corr"].reshape(-1)).sum())
        mg.add_ints("correspondences", m, bad)
        assert bad == 0, f"{config} factor {pick[j]}: {bad} correspondence mismatches"
        off += m
    assert off == len(corr_h)
    mg.save(f"test_full_bench_configuration_sampled[{config}]")


@pytest.mark.parametrize("num,den", [(1, 20), (0, 1), (1, 1)])
def test_linearize_select_equals_two_calls(gv, ctx, num, den):
    """gvox_linearize_batch_accum_select (decisions stay on the device, the
    batch is compacted there) gives bitwise the records of gvox_overlap_select
    to the host + gvox_linearize_batch_accum over the selected list, including
    all / none selected, and repeated calls are bitwise reproducible."""
    import torch
    sc = synth.make("C5", n_submaps=48, half_blocks=4)
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, clouds, sc.r0, sc.levels)
    cand = np.zeros(len(sc.pairs), gv.FACTOR_DTYPE)
    for i, name in enumerate(("source_cloud", "target_map", "pose_i", "pose_j")):
        cand[name] = sc.pairs[:, i]
    sel = gv.overlap_select(ctx, clouds, maps, sc.pairs, sc.poses, sc.overlap_level, num, den)
    fac = cand[sel.view(bool)]
    dsel = torch.from_numpy(sel).cuda()
    out = gv.device_records(ctx, len(cand), gv.FACTOR_ACCUM_DTYPE)
    sel_h = np.full(len(cand), 7, np.uint8)
    ns = gv.linearize_batch_accum_select(ctx, clouds, maps, cand, dsel, sc.poses, out,
                                         selected_host=sel_h)
    assert ns == len(fac) and np.array_equal(sel_h, sel)
    if num == 1 and den == 1:
        assert ns == 0
    if ns:
        ref = gv.device_records(ctx, ns, gv.FACTOR_ACCUM_DTYPE)
        gv.linearize_batch_accum(ctx, clouds, maps, fac, sc.poses, out=ref)
        assert torch.equal(out[:ns], ref)
        out2 = gv.device_records(ctx, len(cand), gv.FACTOR_ACCUM_DTYPE)
        assert gv.linearize_batch_accum_select(ctx, clouds, maps, cand, dsel, sc.poses, out2) == ns
        assert torch.equal(out2[:ns], out[:ns])
    # errors: a candidate out of range, no candidates
    bad = cand.copy()
    bad["target_map"][0] = len(maps)
    with pytest.raises(gv.GvoxError):
        gv.linearize_batch_accum_select(ctx, clouds, maps, bad, dsel, sc.poses, out)
    assert gv.linearize_batch_accum_select(ctx, clouds, maps, cand[:0], dsel, sc.poses, out) == 0


def test_linearize_select_variant_from_selected(gv, ctx, monkeypatch):
    """The screened batch picks its kernel variant from the SELECTED candidates
    (class bits reduced on the device during the compaction), as
    gvox_linearize_batch_accum would for the selected list: unselected
    candidates on a 2-level map and on a hash-level map leave the batch on the
    FAST all-dense kernel; selecting the 2-level one switches it to the generic
    kernel, selecting the hash-level one to the FAST hash-level kernel.  Records
    bitwise the two-call path's either way."""
    import torch
    sc = synth.make("C5", n_submaps=24, half_blocks=3)
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, clouds, sc.r0, sc.levels)
    t0 = int(sc.pairs[0, 1])
    two = gv.create_voxelmap(ctx, clouds[t0], sc.r0, 2)
    monkeypatch.setenv("GVOX_DENSE_BUDGET_MB", "0")
    hashed = gv.create_voxelmap(ctx, clouds[t0], sc.r0, sc.levels)
    monkeypatch.delenv("GVOX_DENSE_BUDGET_MB")
    allm = list(maps) + [two, hashed]
    cand = np.zeros(len(sc.pairs) + 2, gv.FACTOR_DTYPE)
    for i, name in enumerate(("source_cloud", "target_map", "pose_i", "pose_j")):
        cand[name][:-2] = sc.pairs[:, i]
        cand[name][-2:] = sc.pairs[0, i]
    cand["target_map"][-2:] = [len(maps), len(maps) + 1]
    sel = np.zeros(len(cand), np.uint8)
    sel[:-2] = gv.overlap_select(ctx, clouds, maps, sc.pairs, sc.poses, sc.overlap_level, 1, 20)
    assert sel.sum() > 0
    FAST, DENSE = 1, 2
    for extra, want_fast in ((None, True), (-2, False), (-1, True)):
        s = sel.copy()
        if extra is not None:
            s[extra] = 1
        out = gv.device_records(ctx, len(cand), gv.FACTOR_ACCUM_DTYPE)
        ns = gv.linearize_batch_accum_select(ctx, clouds, allm, cand, torch.from_numpy(s).cuda(),
                                             sc.poses, out)
        v = gv.last_linearize_variant()
        assert ns == int(s.sum())
        assert bool(v & FAST) == want_fast, (extra, v)
        assert bool(v & DENSE) == (extra != -1), (extra, v)
        ref = gv.device_records(ctx, ns, gv.FACTOR_ACCUM_DTYPE)
        gv.linearize_batch_accum(ctx, clouds, allm, cand[s.view(bool)], sc.poses, out=ref)
        assert gv.last_linearize_variant() == v
        assert torch.equal(out[:ns], ref)


def test_exec_order_by_target_is_bitwise_neutral(gv, ctx, monkeypatch):
    """GVOX_LIN_EXEC_ORDER=1 executes the tiles grouped by target map (device
    counting sort in the screened batch, host sort in gvox_linearize_batch for
    batches of more than 4096 tiles): the records are bitwise those of the
    batch order."""
    import torch
    sc = synth.make("C5", n_submaps=96, half_blocks=5)
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, clouds, sc.r0, sc.levels)
    cand = np.zeros(len(sc.pairs), gv.FACTOR_DTYPE)
    for i, name in enumerate(("source_cloud", "target_map", "pose_i", "pose_j")):
        cand[name] = sc.pairs[:, i]
    sel = gv.overlap_select(ctx, clouds, maps, sc.pairs, sc.poses, sc.overlap_level, 1, 20)
    dsel = torch.from_numpy(sel).cuda()
    fac = cand[sel.view(bool)]
    res = {}
    for eo in ("0", "1"):
        monkeypatch.setenv("GVOX_LIN_EXEC_ORDER", eo)
        out = gv.device_records(ctx, len(cand), gv.FACTOR_ACCUM_DTYPE)
        ns = gv.linearize_batch_accum_select(ctx, clouds, maps, cand, dsel, sc.poses, out)
        full = gv.linearize_batch(ctx, clouds, maps, cand, sc.poses)  # every candidate: > 4096 tiles
        res[eo] = (ns, out[:ns].clone(), full)
    monkeypatch.delenv("GVOX_LIN_EXEC_ORDER")
    assert res["0"][0] == res["1"][0] == len(fac)
    assert torch.equal(res["0"][1], res["1"][1])
    assert res["0"][2].tobytes() == res["1"][2].tobytes()


def test_dense_and_hash_levels_agree(gv, ctx, monkeypatch):
    """The two voxel index structures (dense grids, hash tables) give identical
    maps and bitwise identical linearizations and overlap counts: the build is
    forced to hash every level with a zero dense budget."""
    sc = synth.global_scene(n_submaps=6, n_points=20000, half_blocks=2, factor_dist=40.0,
                            cand_dist=60.0)
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    f = sc.factors.copy()
    f[:, 4] = 0
    dense = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    monkeypatch.setenv("GVOX_DENSE_BUDGET_MB", "0")
    hashed = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    monkeypatch.delenv("GVOX_DENSE_BUDGET_MB")
    for m1, m2 in zip(dense, hashed):
        for l in range(sc.levels):
            a, b = m1.export(ctx, l), m2.export(ctx, l)
            for x, y in zip(a, b):
                assert np.array_equal(x, y)
    r1 = gv.linearize_batch(ctx, clouds, dense, f, sc.poses)
    r2 = gv.linearize_batch(ctx, clouds, hashed, f, sc.poses)
    assert r1.tobytes() == r2.tobytes()
    c1 = gv.overlap(ctx, clouds, dense, sc.pairs, sc.poses, sc.overlap_level)
    c2 = gv.overlap(ctx, clouds, hashed, sc.pairs, sc.poses, sc.overlap_level)
    assert np.array_equal(c1, c2)


def test_recycled_grid_arena_is_clean(gv, ctx):
    """Dense index grids are recycled (gvox_runtime.cu GridArena): when the
    last map of a build goes, exactly its voxels' cells are reset to -1 and the
    arena serves the next build without a fill.  A build into a recycled arena
    -- including one that previously held OTHER clouds -- gives the maps and
    results of a build into a fresh one (a new context: empty pool)."""
    import gc
    sc = synth.global_scene(n_submaps=6, n_points=20000, half_blocks=2, factor_dist=40.0,
                            cand_dist=60.0)
    f = sc.factors.copy()
    f[:, 4] = 0
    shifted = sc.mu + np.float32(3.3)  # other cells, same sizes -> same arena size class
    fresh = gv.Context(0)
    c_ref = [gv.Cloud(fresh, *sc.cloud(c)) for c in range(sc.num_clouds)]
    m_ref = gv.create_voxelmaps(fresh, [c_ref[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    r_ref = gv.linearize_batch(fresh, c_ref, m_ref, f, sc.poses)
    o_ref = gv.overlap(fresh, c_ref, m_ref, sc.pairs, sc.poses, sc.overlap_level)
    k = gv.Context(0)
    clouds = [gv.Cloud(k, *sc.cloud(c)) for c in range(sc.num_clouds)]
    other = [gv.Cloud(k, shifted[sc.offsets[c]:sc.offsets[c + 1]], *sc.cloud(c)[1:])
             for c in range(sc.num_clouds)]
    for rnd in range(3):
        tmp = gv.create_voxelmaps(k, [other[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
        del tmp
        gc.collect()                       # -> reset + parked in the pool
        maps = gv.create_voxelmaps(k, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
        for a, b in zip(maps, m_ref):
            for l in range(sc.levels):
                for x, y in zip(a.export(k, l), b.export(fresh, l)):
                    assert np.array_equal(x, y)
        assert gv.linearize_batch(k, clouds, maps, f, sc.poses).tobytes() == r_ref.tobytes()
        assert np.array_equal(gv.overlap(k, clouds, maps, sc.pairs, sc.poses, sc.overlap_level), o_ref)
        del maps
        gc.collect()


@pytest.mark.parametrize("hash_levels", [False, True])
def test_sync_free_build_equals_counted(gv, ctx, monkeypatch, hash_levels):
    """Small chunks build sync-free (buffers sized by one voxel per point and
    level, accumulators zeroed by the insert, counts left on the device until
    asked); the counted build (one count readback, exact sizes) gives the same
    maps and bitwise the same linearization, with dense grids and with hash
    levels; the range error is raised by the host box test either way."""
    sc = synth.make("C2")
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    if hash_levels:
        monkeypatch.setenv("GVOX_DENSE_BUDGET_MB", "0")
    monkeypatch.setenv("GVOX_BUILD_NOSYNC", "1")
    fast = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    monkeypatch.setenv("GVOX_BUILD_NOSYNC", "0")
    counted = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    monkeypatch.delenv("GVOX_BUILD_NOSYNC")
    for a, b in zip(fast, counted):
        for l in range(sc.levels):
            assert a.num_voxels(l) == b.num_voxels(l) > 0
            for x, y in zip(a.export(ctx, l), b.export(ctx, l)):
                assert np.array_equal(x, y)
    r1 = gv.linearize_batch(ctx, clouds, fast, sc.factors, sc.poses)
    r2 = gv.linearize_batch(ctx, clouds, counted, sc.factors, sc.poses)
    assert r1.tobytes() == r2.tobytes()
    far = gv.Cloud(ctx, np.array([[0, 0, 0], [2.5e6, 0, 0]], np.float32), np.ones((2, 6), np.float32))
    for flag in ("0", "1"):
        monkeypatch.setenv("GVOX_BUILD_NOSYNC", flag)
        with pytest.raises(gv.GvoxError, match="GVOX_ERR_RANGE"):
            gv.create_voxelmap(ctx, far, 1.0, 1)


@pytest.mark.parametrize("nosync", ["0", "1"])
def test_lifted_accumulation_equals_direct(gv, ctx, monkeypatch, nosync):
    """Lifted builds (level 0 accumulated from the points, every coarser level
    from the voxels below it -- large chunks by default) and direct builds
    (every level from the points) give the same voxels and counts bit for bit
    and the same statistics up to the fixed-point scale (one scale for every
    level vs one per level: ~2^-40 r), for counted and sync-free builds."""
    sc = synth.global_scene(n_submaps=6, n_points=20000, half_blocks=2, factor_dist=40.0,
                            cand_dist=60.0)
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    monkeypatch.setenv("GVOX_BUILD_NOSYNC", nosync)
    out = {}
    for lift in ("1", "0"):
        monkeypatch.setenv("GVOX_BUILD_LIFT", lift)
        out[lift] = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    for a, b in zip(out["1"], out["0"]):
        for l in range(sc.levels):
            ka, ma, ca, na = a.export(ctx, l)
            kb, mb, cb, nb = b.export(ctx, l)
            assert np.array_equal(ka, kb) and np.array_equal(na, nb)
            r = sc.r0 * 2 ** l
            np.testing.assert_allclose(ma, mb, rtol=0, atol=1e-6 * r)
            np.testing.assert_allclose(ca, cb, rtol=0, atol=1e-6 * np.abs(cb).max())
    f = sc.factors.copy()
    f[:, 4] = 0
    r1 = gv.linearize_batch(ctx, clouds, out["1"], f, sc.poses)
    r0 = gv.linearize_batch(ctx, clouds, out["0"], f, sc.poses)
    assert np.array_equal(r1["inliers"], r0["inliers"])
    np.testing.assert_allclose(r1["error"], r0["error"], rtol=1e-5)
