"""GPU preprocessing (gvox_knn, gvox_estimate_covariances; P:186, P:262;
SURVEY §8(f) NEXT-3) vs the oracle (oracle/preprocess.py).

Bars: neighbour tables bit-exact (integers, unique by reading R26); the
regularized covariance within 2e-6 absolute (fp32 output of fp64 arithmetic)
wherever the neighbourhood's smallest eigenvalue is separated from the next
by more than 1e-4 of the largest (elsewhere the normal is ill-conditioned
or not unique: the result is checked for validity instead); normals equal up
to the orientation rule's sign, which must match wherever |n . mu| is not
tiny.  Edge cases: empty and one-point clouds, short rows (n < k), duplicate
points (ties by index), k = 1 and k = 20 (the 32-wide kernel), cell sizes
that change the search but never the result, a full C3 batch checked on
sampled rows."""
import numpy as np
import pytest

import synth
from oracle import preprocess as pp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(gv):
    return gv.Context(0)


def lidar_cloud(n, seed=2):
    sc = synth.odometry_step(n_kf=1, n_points=n, rings=64, az=512, seed=seed)
    return sc.cloud(0)[0]


def check_cov(pts, nb, cov, nrm):
    ocov, onrm = pp.covariances(pts, nb)
    P = pts.astype(np.float64)
    bad = 0
    for i in range(len(pts)):
        sel = nb[i][nb[i] >= 0]
        D = P[sel] - P[sel].mean(0)
        S = D.T @ D / len(sel)
        w = np.linalg.eigvalsh(S)
        if w[2] == 0:
            np.testing.assert_array_equal(cov[i], np.float32([1e-6, 0, 0, 1e-6, 0, 1e-6]))
            assert not nrm[i].any()
            continue
        if (w[1] - w[0]) > 1e-4 * w[2]:
            np.testing.assert_allclose(cov[i], ocov[i], atol=2e-6, rtol=0)
            if abs(onrm[i] @ P[i]) > 1e-3 * np.linalg.norm(P[i]):
                np.testing.assert_allclose(nrm[i], onrm[i], atol=2e-6)
        else:  # validity: a unit eigenvector of the smallest eigenvalue, oriented
            bad += 1
            n = nrm[i].astype(np.float64)
            assert abs(np.linalg.norm(n) - 1) < 1e-6
            assert np.linalg.norm(S @ n - w[0] * n) <= 1e-5 * w[2] + 1e-12
            assert n @ P[i] <= 1e-6 * np.linalg.norm(P[i])
    return bad


@pytest.mark.parametrize("k,cell", [(10, 0.5), (1, 0.5), (20, 0.5), (10, 0.05), (10, 5.0)])
def test_knn_lidar_frame(gv, ctx, k, cell):
    pts = lidar_cloud(4000)
    got = gv.knn(ctx, pts, k=k, cell_size=cell)
    ref = pp.knn(pts, k)
    assert np.array_equal(got, ref)


def test_knn_batch_edge_cases_and_covariances(gv, ctx):
    rs = np.random.default_rng(1)
    a = (rs.normal(0, 4, (2500, 3)) * [1, 1, 0.1]).astype(np.float32)
    dup = np.repeat(rs.uniform(-1, 1, (30, 3)).astype(np.float32), 3, axis=0)  # exact duplicates
    one = np.float32([[1.0, 2.0, 3.0]])
    five = rs.uniform(-1, 1, (5, 3)).astype(np.float32)
    line = np.c_[np.linspace(0, 3, 40), np.zeros(40), np.zeros(40)].astype(np.float32) + [0, 1, 0]
    clouds = [a, np.zeros((0, 3), np.float32), dup, one, five, line]
    pts = np.concatenate(clouds)
    off = np.cumsum([0] + [len(c) for c in clouds])
    k = 10
    got = gv.knn(ctx, pts, k=k, cell_size=0.3, offsets=off)
    for c, cl in enumerate(clouds):
        ref = pp.knn(cl, k) if len(cl) else np.zeros((0, k), np.int32)
        assert np.array_equal(got[off[c]:off[c + 1]], ref), c
    cov, nrm = gv.estimate_covariances(ctx, pts, got, offsets=off)
    for c, cl in enumerate(clouds):
        if len(cl):
            check_cov(cl, got[off[c]:off[c + 1]], cov[off[c]:off[c + 1]], nrm[off[c]:off[c + 1]])
    # device tensors give the same tables
    import torch
    tp = torch.from_numpy(pts).cuda()
    dnb = gv.knn(ctx, tp, k=k, cell_size=0.3, offsets=off)
    dcov, dnrm = gv.estimate_covariances(ctx, tp, dnb, offsets=off)
    torch.cuda.synchronize()
    assert np.array_equal(dnb.cpu().numpy(), got)
    assert np.array_equal(dcov.cpu().numpy(), cov) and np.array_equal(dnrm.cpu().numpy(), nrm)
    with pytest.raises(gv.GvoxError):
        bad = got.copy()
        bad[0, 0] = 10 ** 6
        gv.estimate_covariances(ctx, pts, bad, offsets=off)
    with pytest.raises(gv.GvoxError):
        gv.knn(ctx, pts, k=33, offsets=off)


def test_covariances_lidar_frame(gv, ctx):
    pts = lidar_cloud(3000, seed=5)
    nb = gv.knn(ctx, pts, k=10)
    cov, nrm = gv.estimate_covariances(ctx, pts, nb)
    bad = check_cov(pts, nb, cov, nrm)
    assert bad < len(pts) // 20


def test_full_c3_batch_sampled(gv, ctx):
    sc = synth.make("C3")
    pts = sc.mu
    off = sc.offsets
    nb = gv.knn(ctx, pts, k=10, cell_size=0.5, offsets=off)
    rs = np.random.default_rng(0)
    for c in rs.choice(sc.num_clouds, 5, replace=False):
        cl = pts[off[c]:off[c + 1]]
        for i in rs.choice(len(cl), 40, replace=False):
            d2 = pp.sq_dist(cl[i], cl)
            ref = np.lexsort((np.arange(len(cl)), d2))[:10]
            assert nb[off[c] + i].tolist() == ref.tolist()


@pytest.mark.parametrize("k", [1, 10, 16])
def test_knn_lanes_per_query_agree(gv, ctx, monkeypatch, k):
    """The k-NN query with 1, 4, 8 or 16 lanes per query (GVOX_KNN_GROUP; the
    library picks 4 for small batches, 1 for large ones) returns bitwise the
    same tables -- each is checked against the brute-force oracle too."""
    pts = lidar_cloud(6000, seed=5)
    want = pp.knn(pts, k)
    got = {}
    for g in ("1", "4", "8", "16"):
        monkeypatch.setenv("GVOX_KNN_GROUP", g)
        got[g] = gv.knn(ctx, pts, k, cell_size=0.5)
        assert np.array_equal(got[g], want), f"G = {g}"
    monkeypatch.delenv("GVOX_KNN_GROUP")
    assert np.array_equal(gv.knn(ctx, pts, k, cell_size=0.5), want)
