"""Oracle of the global Gauss-Newton step (gvox_solve_global; SURVEY §8(f)
NEXT-4; global mapping P:391, solver P:814).

TEST INFRASTRUCTURE ONLY (imported by tests/).  Plain numpy, dense, fp64:

  variables = the poses not fixed, in pose order;
  for every factor f (pose_i, pose_j) with the oracle's full 12x12 H_f and
  12-vector b_f (Eqs. 4-8, oracle.cpp, no adjoint shortcut):
      H[i,i] += H_ii,  H[j,j] += H_jj,  H[i,j] += H_ij,  H[j,i] += H_ij^T,
      b[i] += b_i,     b[j] += b_j        (terms of fixed poses dropped);
  H += lambda I;  delta = solve(H, -b)  (numpy LAPACK).
"""
from __future__ import annotations

import numpy as np


def assemble(factors, lin, num_poses, fixed, lam=0.0):
    factors = np.asarray(factors, np.int64).reshape(-1, 5)
    var = -np.ones(num_poses, np.int64)
    nv = 0
    for p in range(num_poses):
        if not fixed[p]:
            var[p] = nv
            nv += 1
    H = np.zeros((6 * nv, 6 * nv))
    b = np.zeros(6 * nv)
    for f in range(len(factors)):
        vi, vj = var[factors[f, 2]], var[factors[f, 3]]
        Hf, bf = lin[f]["H"], lin[f]["b"]
        si, sj = slice(6 * vi, 6 * vi + 6), slice(6 * vj, 6 * vj + 6)
        if vi >= 0:
            H[si, si] += Hf[:6, :6]
            b[si] += bf[:6]
        if vj >= 0:
            H[sj, sj] += Hf[6:, 6:]
            b[sj] += bf[6:]
        if vi >= 0 and vj >= 0:
            H[si, sj] += Hf[:6, 6:]
            H[sj, si] += Hf[6:, :6]
    H += lam * np.eye(6 * nv)
    return H, b, var


def solve(H, b):
    return np.linalg.solve(H, -b)
