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


def optimize(clouds, maps, factors, poses, fixed, max_iterations=10, lam=0.0, eps_rot=1e-6,
             eps_trans=1e-6, num_threads=1):
    """Gauss-Newton over the whole graph (P:391 global mapping; every factor
    re-linearized each iteration): linearize all factors (oracle.cpp),
    assemble, solve, T_v <- T_v Exp(delta_v) for the variables; stop when the
    largest |w| and |rho| of a step are within eps.  Returns (poses, errors,
    converged)."""
    from . import oracle as _o
    from .register import se3_exp
    poses = np.array(np.asarray(poses, np.float64).reshape(-1, 12))
    P = len(poses)
    errs = []
    for _ in range(max_iterations):
        lin = _o.linearize_batch(clouds, maps, factors, poses, num_threads=num_threads)
        errs.append(sum(d["e"] for d in lin))
        H, b, var = assemble(factors, lin, P, fixed, lam)
        x = solve(H, b)
        mw = mr = 0.0
        for v in range(P):
            if var[v] < 0:
                continue
            d = x[6 * var[v]: 6 * var[v] + 6]
            mw, mr = max(mw, float(np.linalg.norm(d[:3]))), max(mr, float(np.linalg.norm(d[3:])))
            T = np.eye(4)
            T[:3, :] = poses[v].reshape(3, 4)
            poses[v] = (T @ se3_exp(d))[:3, :].reshape(12)
        if mw <= eps_rot and mr <= eps_trans:
            return poses, errs, True
    return poses, errs, False
