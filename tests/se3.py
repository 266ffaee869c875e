"""Test-local SE(3) helpers (rotation-first tangent [w; rho], right perturbation
T <- T Exp(xi)).  Independent of both the oracle and the CUDA path."""
import math

import numpy as np


def hat(w):
    return np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0.0]])


def so3_exp(w):
    th = float(np.linalg.norm(w))
    K = hat(w)
    if th < 1e-9:
        return np.eye(3) + K + 0.5 * K @ K
    return np.eye(3) + math.sin(th) / th * K + (1 - math.cos(th)) / th ** 2 * (K @ K)


def se3_exp(xi):
    w, rho = np.asarray(xi[:3], float), np.asarray(xi[3:], float)
    th = float(np.linalg.norm(w))
    K = hat(w)
    if th < 1e-9:
        V = np.eye(3) + 0.5 * K + K @ K / 6.0
    else:
        V = np.eye(3) + (1 - math.cos(th)) / th ** 2 * K + (th - math.sin(th)) / th ** 3 * (K @ K)
    T = np.eye(4)
    T[:3, :3] = so3_exp(w)
    T[:3, 3] = V @ rho
    return T


def to44(T12):
    T = np.eye(4)
    T[:3, :] = np.asarray(T12, float).reshape(3, 4)
    return T


def to12(T44):
    return np.ascontiguousarray(T44[:3, :].reshape(12))


def right_perturb(T12, xi):
    return to12(to44(T12) @ se3_exp(xi))


def adjoint(T12):
    """Ad(T) for rotation-first tangents: [[R, 0], [t^ R, R]]."""
    T = np.asarray(T12, float).reshape(3, 4)
    R, t = T[:, :3], T[:, 3]
    Ad = np.zeros((6, 6))
    Ad[:3, :3] = R
    Ad[3:, 3:] = R
    Ad[3:, :3] = hat(t) @ R
    return Ad


def random_pose(rs, rot_scale=1.0, trans_scale=5.0):
    R = so3_exp(rs.normal(0, rot_scale, 3))
    T = np.eye(4)
    T[:3, :3] = R
    T[:3, 3] = rs.normal(0, trans_scale, 3)
    return to12(T)


def rel_pose(Ti, Tj):
    """T_j^-1 T_i in plain numpy (for tests only)."""
    return to12(np.linalg.inv(to44(Tj)) @ to44(Ti))


def plane_cov(n, eps=1e-3):
    n = np.asarray(n, float) / np.linalg.norm(n)
    C = np.eye(3) - (1 - eps) * np.outer(n, n)
    return np.array([C[0, 0], C[0, 1], C[0, 2], C[1, 1], C[1, 2], C[2, 2]])


def cov6_to33(c):
    c = np.asarray(c, float)
    return np.array([[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]])
