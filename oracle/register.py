"""Oracle of the on-device registration loop (gvox_register_batch, SURVEY
§8(f) NEXT-1): plain fp64 numpy Gauss-Newton over independent variable poses.

TEST INFRASTRUCTURE ONLY: imported by tests/ and the registration bench's
cpu_baseline leg.  The product package never imports it.

What it follows:
  * Omega is fixed at the linearization point, so each iteration is a
    weighted least-squares (Gauss-Newton) step on e^PC (Eq. 2);
  * "we re-evaluate each matching cost factor ... in each optimization
    iteration": every iteration re-linearizes every factor (new
    correspondences, new Omega) at the current poses;
  * Eqs. 4-8 — H_ii and b_i of each factor, taken here from the
    oracle's full 12x12 J^T Omega J (oracle.cpp, no adjoint shortcut);
  * right perturbation T <- T Exp(delta), rotation-first delta = [w; rho]
    (include/gvox.h conventions, reading Q1/Q4): e(delta) ~ e + 2 b^T delta +
    delta^T H delta, minimised by (H + lambda I) delta = -b (lambda = 0: GN).
Per variable pose v: H = sum_f H_ii(f), b = sum_f b_i(f), e = sum_f e(f) over
the factors with pose_i = v, in ascending factor order; Cholesky (numpy)
decides "singular"; stop when |w| <= eps_rot and |rho| <= eps_trans, or after
max_iterations linearizations.
"""
from __future__ import annotations

import math

import numpy as np

from . import oracle as _o

REG_FIXED, REG_MAX_ITER, REG_CONVERGED, REG_SINGULAR = 0, 1, 2, 3


def hat(w):
    return np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])


def se3_exp(xi):
    """Exp of the twist [w; rho] as a 4x4 matrix, closed form:
    R = I + A W + B W^2, t = (I + B W + C W^2) rho with W = w^,
    A = sin(th)/th, B = (1 - cos th)/th^2, C = (th - sin th)/th^3
    (series below th = 1e-4).  Pinned against scipy.linalg.expm of the 4x4
    twist matrix in tests/test_oracle_register.py."""
    xi = np.asarray(xi, np.float64)
    w, rho = xi[:3], xi[3:]
    th2 = float(w @ w)
    th = math.sqrt(th2)
    if th < 1e-4:
        A = 1.0 - th2 / 6.0 + th2 * th2 / 120.0
        B = 0.5 - th2 / 24.0 + th2 * th2 / 720.0
        C = 1.0 / 6.0 - th2 / 120.0 + th2 * th2 / 5040.0
    else:
        A = math.sin(th) / th
        B = (1.0 - math.cos(th)) / th2
        C = (th - math.sin(th)) / (th2 * th)
    W = hat(w)
    W2 = W @ W
    T = np.eye(4)
    T[:3, :3] = np.eye(3) + A * W + B * W2
    T[:3, 3] = (np.eye(3) + B * W + C * W2) @ rho
    return T


def register_batch(clouds, maps, factors, poses, max_iterations=10, lam=0.0, eps_rot=1e-6,
                   eps_trans=1e-6, num_threads=1):
    """clouds: list of (mu, cov, normals|None); maps: list of oracle.VoxelMap;
    factors int64 [F,5] {source, target, pose_i (variable), pose_j (fixed), flags};
    poses [P,12].  Returns (poses_out [P,12], results list of dicts indexed by
    pose, history [max_iterations, P])."""
    factors = np.asarray(factors, np.int64).reshape(-1, 5)
    poses = np.array(np.asarray(poses, np.float64).reshape(-1, 12))
    P = poses.shape[0]
    var = sorted(set(int(v) for v in factors[:, 2]))
    assert not (set(int(j) for j in factors[:, 3]) & set(var)), "pose_j must be fixed"
    results = [dict(status=REG_FIXED, iterations=0, inliers=0, error_initial=0.0,
                    error_final=0.0, last_step=np.zeros(6)) for _ in range(P)]
    for v in var:
        results[v]["status"] = REG_MAX_ITER
    history = np.zeros((max_iterations, P))
    active = list(var)
    for k in range(max_iterations):
        if not active:
            break
        rows = [f for f in range(len(factors)) if int(factors[f, 2]) in active]
        lin = _o.linearize_batch(clouds, maps, factors[rows], poses, num_threads=num_threads)
        by_pose = {v: [] for v in active}
        for idx, f in enumerate(rows):
            by_pose[int(factors[f, 2])].append(lin[idx])  # ascending factor order
        still = []
        for v in active:
            H = np.zeros((6, 6))
            b = np.zeros(6)
            e = 0.0
            inl = 0
            for d in by_pose[v]:
                H += d["H_ii"]
                b += d["b_i"]
                e += d["e"]
                inl += int(d["inliers"].sum())
            r = results[v]
            if k == 0:
                r["error_initial"] = e
            r["error_final"] = e
            r["inliers"] = inl
            r["iterations"] = k + 1
            history[k, v] = e
            try:
                np.linalg.cholesky(H + lam * np.eye(6))
            except np.linalg.LinAlgError:
                r["status"] = REG_SINGULAR
                r["last_step"] = np.zeros(6)
                continue
            delta = np.linalg.solve(H + lam * np.eye(6), -b)
            T = np.eye(4)
            T[:3, :] = poses[v].reshape(3, 4)
            poses[v] = (T @ se3_exp(delta))[:3, :].reshape(12)
            r["last_step"] = delta
            if np.linalg.norm(delta[:3]) <= eps_rot and np.linalg.norm(delta[3:]) <= eps_trans:
                r["status"] = REG_CONVERGED
            elif k + 1 >= max_iterations:
                r["status"] = REG_MAX_ITER
            else:
                still.append(v)
        active = still
    return poses, results, history
