"""Pins of the preprocessing oracle (oracle/preprocess.py; P:186, P:262;
SURVEY §8(f) NEXT-3), CPU only:

* k-NN on hand cases (SPEC knn_search examples: collinear x = 0, 1, 3 with
  k = 2; a one-point cloud; short rows), and against an independent library
  k-d tree (scipy cKDTree): the same sorted distances for every point, the
  same sets wherever no distance tie straddles the k-th place;
* covariances: a coplanar neighbourhood below the sensor gives the upward
  normal; an axis-aligned anisotropic neighbourhood gives its thinnest axis;
  the regularized covariance has eigenvalues (1e-3, 1, 1) with the normal as
  the 1e-3 eigenvector; coincident neighbours give 1e-6 I and a zero normal.
"""
import numpy as np
import scipy.spatial

from oracle import preprocess as pp


def test_knn_hand_cases():
    pts = np.array([[0, 0, 0], [1, 0, 0], [3, 0, 0]], np.float32)
    nb = pp.knn(pts, 2)
    assert nb[1].tolist() == [1, 0]
    assert nb[0].tolist() == [0, 1] and nb[2].tolist() == [2, 1]
    assert pp.knn(pts[:1], 1).tolist() == [[0]]
    short = pp.knn(pts, 5)
    assert short[1].tolist() == [1, 0, 2, -1, -1]
    # equal distances: the smaller index first
    sq = np.array([[0, 0, 0], [1, 0, 0], [-1, 0, 0], [0, 1, 0]], np.float32)
    assert pp.knn(sq, 4)[0].tolist() == [0, 1, 2, 3]


def test_knn_matches_kdtree():
    rs = np.random.default_rng(4)
    pts = (rs.normal(0, 5, (1500, 3)) * [1, 1, 0.2]).astype(np.float32)
    k = 10
    nb = pp.knn(pts, k)
    tree = scipy.spatial.cKDTree(pts.astype(np.float64))
    dk, ik = tree.query(pts.astype(np.float64), k=k + 1)
    for i in range(len(pts)):
        d_or = np.sqrt(pp.sq_dist(pts[i], pts[nb[i]]))
        np.testing.assert_allclose(d_or, dk[i, :k], rtol=1e-12, atol=1e-12)
        if dk[i, k] > dk[i, k - 1] * (1 + 1e-9):  # no tie at the k-th place
            assert set(nb[i].tolist()) == set(ik[i, :k].tolist())


def test_covariance_cases():
    rs = np.random.default_rng(9)
    # ground plane 1.5 m below the sensor: normal points up (toward the origin)
    g = np.c_[rs.uniform(2, 4, (10, 2)), np.full(10, -1.5)].astype(np.float32)
    cov, nrm = pp.covariances(g, np.tile(np.arange(10), (10, 1)))
    np.testing.assert_allclose(nrm, np.tile([0, 0, 1.0], (10, 1)), atol=1e-12)
    np.testing.assert_allclose(cov[0], [1, 0, 0, 1, 0, 1e-3], atol=1e-12)
    # anisotropic, axis-aligned: thinnest axis y; points at x > 0 -> n = -x?  (n . mu <= 0)
    a = (rs.normal(0, 1, (400, 3)) * [3.0, 0.05, 1.0] + [10, 0, 0]).astype(np.float32)
    cov, nrm = pp.covariances(a, np.tile(np.arange(400), (400, 1)))
    assert abs(abs(nrm[0, 1]) - 1) < 1e-3
    for i in range(0, 400, 37):
        assert nrm[i] @ a[i].astype(float) <= 0
        C = np.array([[cov[i, 0], cov[i, 1], cov[i, 2]], [cov[i, 1], cov[i, 3], cov[i, 4]],
                      [cov[i, 2], cov[i, 4], cov[i, 5]]])
        w, U = np.linalg.eigh(C)
        np.testing.assert_allclose(w, [1e-3, 1, 1], atol=1e-12)
        assert abs(abs(U[:, 0] @ nrm[i]) - 1) < 1e-12
    # coincident neighbours
    c = np.ones((5, 3), np.float32)
    cov, nrm = pp.covariances(c, np.tile(np.arange(5), (5, 1)))
    np.testing.assert_array_equal(cov[0], [1e-6, 0, 0, 1e-6, 0, 1e-6])
    np.testing.assert_array_equal(nrm[0], [0, 0, 0])
