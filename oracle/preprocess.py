"""Oracle of the GPU preprocessing: exact k nearest
neighbours and plane-regularized point covariances.

TEST INFRASTRUCTURE ONLY (imported by tests/).  Plain numpy, fp64.

What it follows:
  * "The covariance matrix C_k is calculated from neighboring points of
    p_k given by a k-nearest-neighbor search";
  * "find k neighboring points for each point" ... "the costly EXACT
    nearest neighbor search is only performed in the preprocessing step";
  * SPEC knn_search: the k nearest points by Euclidean distance, self
    included, exact; a cloud with fewer than k points gives short rows.

Readings (R26-R28):
  R26  distance decisions: d2 = (dx*dx + dy*dy) + dz*dz in fp64, each
       operation rounded (no fused multiply-add), dx = float64(x_j) -
       float64(x_i) from the fp32 inputs; neighbours ordered by (d2, index)
       ascending, so the k-set and its order are unique.  Missing entries -1.
  R27  covariance: the k neighbours' sample covariance (mean-centred, / k;
       the scale does not matter below); normal n = unit eigenvector of its
       smallest eigenvalue, oriented toward the cloud origin (n . mu <= 0,
       flipped if n . mu > 0); GICP plane model C = I - (1 - 1e-3) n n^T,
       i.e. eigenvalues (1e-3, 1, 1) on (n, t1, t2) (Segal 2009, the same
       model synth/ uses).
  R28  degenerate neighbourhoods: a zero sample covariance (all neighbours
       coincident, or a single point) gives C = 1e-6 I and n = 0 (SPEC
       "isotropic eps covariance, normal flagged invalid").  When the smallest
       eigenvalue is not simple the normal is not unique: any unit vector of
       its eigenspace is correct (tests check validity, not equality).
"""
from __future__ import annotations

import numpy as np

EPS_PLANE = 1e-3
EPS_DEGENERATE = 1e-6


def sq_dist(p, q):
    """R26: fp64 squared distance with pinned, unfused operation order."""
    d = np.asarray(q, np.float32).astype(np.float64) - np.asarray(p, np.float32).astype(np.float64)
    return (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]


def knn(points, k):
    """Brute force: for each point, the indices of its k nearest points
    (self included) ordered by (d2, index); -1 where the cloud is short."""
    pts = np.asarray(points, np.float32).reshape(-1, 3)
    n = len(pts)
    out = np.full((n, k), -1, np.int32)
    idx = np.arange(n)
    for i in range(n):
        d2 = sq_dist(pts[i], pts)
        order = np.lexsort((idx, d2))[:k]
        out[i, :len(order)] = order
    return out


def covariances(points, neighbors):
    """R27/R28: (cov [n,6] xx xy xz yy yz zz, normals [n,3]) in fp64."""
    pts = np.asarray(points, np.float32).astype(np.float64).reshape(-1, 3)
    nb = np.asarray(neighbors)
    n = len(pts)
    cov = np.zeros((n, 6))
    nrm = np.zeros((n, 3))
    for i in range(n):
        sel = nb[i][nb[i] >= 0]
        P = pts[sel]
        m = P.mean(axis=0)
        D = P - m
        S = D.T @ D / len(sel)
        if not S.any():
            C = EPS_DEGENERATE * np.eye(3)
            v = np.zeros(3)
        else:
            w, U = np.linalg.eigh(S)
            v = U[:, 0]
            if v @ pts[i] > 0:
                v = -v
            C = np.eye(3) - (1.0 - EPS_PLANE) * np.outer(v, v)
        cov[i] = [C[0, 0], C[0, 1], C[0, 2], C[1, 1], C[1, 2], C[2, 2]]
        nrm[i] = v
    return cov, nrm
