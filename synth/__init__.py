"""Seeded synthetic inputs for the VGICP hot path (configs C1..C5 of BASELINE.json).

This module is shared by the oracle side and the CUDA side and contains none of
the method's arithmetic: it produces Gaussian point clouds (mean, covariance,
oriented normal), world poses, factor lists and overlap candidate lists.  The
recipe follows SURVEY.md Sec.8(d) and is restated in DESIGN.md ("Input recipe").

Heavy lifting (ray casting, downsampling) is in gen.cpp (libsynth.so), driven
by a counter-based SplitMix64 generator so results do not depend on threading.
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.cpp")
_LIB = os.path.join(_HERE, "libsynth.so")

WORLD_SEED = 2407_10344
GEN_VERSION = 1


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-shared", "-fPIC", "-pthread", _SRC,
                               "-o", _LIB + ".tmp"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.synth_world_create.restype = P
        L.synth_world_create.argtypes = [ctypes.c_uint64, ctypes.c_int]
        L.synth_world_free.argtypes = [P]
        L.synth_world_occupied.restype = ctypes.c_int
        L.synth_world_occupied.argtypes = [P, ctypes.c_double, ctypes.c_double]
        L.synth_make_clouds.argtypes = [P, ctypes.c_int64, ctypes.c_int, P, P, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int64, ctypes.c_uint64,
                                        ctypes.c_uint64, ctypes.c_int, ctypes.c_int, P, P, P, P]
        _lib = L
    return _lib


def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# small pose helpers (generator-local; 3x4 row-major world <- sensor)
# ---------------------------------------------------------------------------
def _rot_zyx(yaw, pitch, roll):
    cz, sz = math.cos(yaw), math.sin(yaw)
    cy, sy = math.cos(pitch), math.sin(pitch)
    cx, sx = math.cos(roll), math.sin(roll)
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1.0]])
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    return Rz @ Ry @ Rx


def _so3_exp(w):
    th = float(np.linalg.norm(w))
    K = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0.0]])
    if th < 1e-12:
        return np.eye(3) + K
    return np.eye(3) + math.sin(th) / th * K + (1 - math.cos(th)) / th ** 2 * (K @ K)


def _pose(R, t):
    T = np.zeros((3, 4))
    T[:, :3] = R
    T[:, 3] = t
    return T.reshape(12)


def perturb_poses(poses, seed, sigma_t=0.05, sigma_r_deg=0.5):
    """Linearization points: ground truth perturbed by N(0, 5 cm), N(0, 0.5 deg)."""
    rs = np.random.default_rng(seed)
    out = np.empty_like(poses)
    for k in range(poses.shape[0]):
        T = poses[k].reshape(3, 4)
        dR = _so3_exp(rs.normal(0, math.radians(sigma_r_deg), 3))
        dt = rs.normal(0, sigma_t, 3)
        out[k] = _pose(T[:, :3] @ dR, T[:, 3] + dt)
    return out


# ---------------------------------------------------------------------------
# trajectory: random walk on the 40 m street grid
# ---------------------------------------------------------------------------
class StreetPath:
    def __init__(self, seed: int, length_m: float, half_blocks: int, block: float = 40.0):
        rs = np.random.default_rng(seed)
        lim = (half_blocks - 1) * block
        pos = np.array([0.0, 0.0])
        heading = np.array([1.0, 0.0])
        pts = [pos.copy()]
        total = 0.0
        while total < length_m + block:
            opts = []
            left = np.array([-heading[1], heading[0]])
            for h, w in ((heading, 0.5), (left, 0.25), (-left, 0.25)):
                nxt = pos + block * h
                if abs(nxt[0]) <= lim and abs(nxt[1]) <= lim:
                    opts.append((h, w))
            if not opts:
                opts = [(-heading, 1.0)]
            ws = np.array([w for _, w in opts])
            h = opts[int(rs.choice(len(opts), p=ws / ws.sum()))][0]
            pos = pos + block * h
            heading = h
            pts.append(pos.copy())
            total += block
        self.pts = np.array(pts)
        seg = np.linalg.norm(np.diff(self.pts, axis=0), axis=1)
        self.cum = np.concatenate([[0.0], np.cumsum(seg)])
        self.tilt_seed = seed + 17

    def pose(self, s: float, tilt_id: int = 0):
        i = int(np.clip(np.searchsorted(self.cum, s, side="right") - 1, 0, len(self.pts) - 2))
        a, b = self.pts[i], self.pts[i + 1]
        u = (s - self.cum[i]) / max(self.cum[i + 1] - self.cum[i], 1e-9)
        p = a + u * (b - a)
        yaw = math.atan2(b[1] - a[1], b[0] - a[0])
        rs = np.random.default_rng([self.tilt_seed, tilt_id])
        pitch, roll = rs.normal(0, math.radians(1.0), 2)
        z = 1.5 + rs.normal(0, 0.02)
        return _pose(_rot_zyx(yaw, pitch, roll), np.array([p[0], p[1], z]))


# ---------------------------------------------------------------------------
# scenes
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class Scene:
    name: str
    mu: np.ndarray        # float32 [Ntot,3], clouds concatenated
    cov: np.ndarray       # float32 [Ntot,6] xx xy xz yy yz zz
    nrm: np.ndarray       # float32 [Ntot,3]
    offsets: np.ndarray   # int64 [C+1]
    map_clouds: np.ndarray  # int64 [M]: cloud each voxel map is built from
    r0: float
    levels: int
    factors: np.ndarray   # int64 [F,5] {source cloud, target map, pose_i, pose_j, flags}
    poses: np.ndarray     # float64 [P,12] linearization points (world <- sensor)
    gt_poses: np.ndarray  # float64 [P,12]
    pairs: np.ndarray     # int64 [Q,4] overlap candidates {source cloud, target map, pose_i, pose_j}
    overlap_level: int

    @property
    def num_clouds(self):
        return len(self.offsets) - 1

    def cloud(self, c):
        a, b = int(self.offsets[c]), int(self.offsets[c + 1])
        return self.mu[a:b], self.cov[a:b], self.nrm[a:b]

    def cloud_size(self, c):
        return int(self.offsets[c + 1] - self.offsets[c])

    @property
    def point_factors(self):
        n = np.diff(self.offsets)
        return int(n[self.factors[:, 0]].sum()) if len(self.factors) else 0


def _make_clouds(world, frame_poses, origin_poses, fpc, rings, az, ds_res, n_target, seed,
                 first_id, order_random=False, threads=None):
    C = origin_poses.shape[0]
    mu = np.zeros((C * n_target, 3), np.float32)
    cov = np.zeros((C * n_target, 6), np.float32)
    nrm = np.zeros((C * n_target, 3), np.float32)
    counts = np.zeros(C, np.int64)
    fp = np.ascontiguousarray(frame_poses, np.float64)
    op = np.ascontiguousarray(origin_poses, np.float64)
    lib().synth_make_clouds(world, C, fpc, fp.ctypes.data, op.ctypes.data, rings, az, 60.0, 0.01,
                            ds_res, n_target, seed, first_id, int(order_random),
                            threads or host_threads(), mu.ctypes.data, cov.ctypes.data,
                            nrm.ctypes.data, counts.ctypes.data)
    # compact (clouds with fewer cells than n_target)
    if np.all(counts == n_target):
        offsets = np.arange(C + 1, dtype=np.int64) * n_target
        return mu, cov, nrm, offsets
    keep = np.concatenate([np.arange(c * n_target, c * n_target + counts[c]) for c in range(C)])
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return mu[keep], cov[keep], nrm[keep], offsets


class _World:
    def __init__(self, half_blocks, seed=WORLD_SEED):
        self.h = lib().synth_world_create(seed, half_blocks)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.synth_world_free(self.h)
            self.h = None


def room_corner(seed=1, n=1000):
    """C1: 1k-point room-corner scene (floor + 3 walls), source = an independent
    resample under a known pose; r = 1.0 m, L = 1 (one factor)."""
    rs = np.random.default_rng(seed)

    def sample(m, rsi):
        # planes: floor z=0 (6x6), wall x=0 (6x3), wall y=0 (6x3), wall x=6 (6x3)
        areas = np.array([36.0, 18.0, 18.0, 18.0])
        which = rsi.choice(4, size=m, p=areas / areas.sum())
        u = rsi.uniform(0, 1, m)
        v = rsi.uniform(0, 1, m)
        p = np.zeros((m, 3))
        nv = np.zeros((m, 3))
        f = which == 0
        p[f] = np.stack([6 * u[f], 6 * v[f], 0 * u[f]], 1); nv[f] = [0, 0, 1]
        f = which == 1
        p[f] = np.stack([0 * u[f], 6 * u[f], 3 * v[f]], 1); nv[f] = [1, 0, 0]
        f = which == 2
        p[f] = np.stack([6 * u[f], 0 * u[f], 3 * v[f]], 1); nv[f] = [0, 1, 0]
        f = which == 3
        p[f] = np.stack([6 + 0 * u[f], 6 * u[f], 3 * v[f]], 1); nv[f] = [-1, 0, 0]
        p += nv * rsi.normal(0, 0.01, (m, 1))
        nj = nv + rsi.normal(0, 0.02, (m, 3))
        nj /= np.linalg.norm(nj, axis=1, keepdims=True)
        e = 1 - 1e-3
        C = np.stack([1 - e * nj[:, 0] ** 2, -e * nj[:, 0] * nj[:, 1], -e * nj[:, 0] * nj[:, 2],
                      1 - e * nj[:, 1] ** 2, -e * nj[:, 1] * nj[:, 2], 1 - e * nj[:, 2] ** 2], 1)
        return p, C, nj

    pt, Ct, nt = sample(n, rs)
    ps, Cs, ns = sample(n, rs)
    # target frame = world; source sensor pose (known) inside the room
    T_s = _pose(_rot_zyx(0.3, 0.02, -0.01), np.array([2.5, 3.0, 1.2]))
    R = T_s.reshape(3, 4)[:, :3]
    t = T_s.reshape(3, 4)[:, 3]
    ps_local = (ps - t) @ R            # R^T (p - t)
    ns_local = ns @ R
    Cs_m = np.zeros((n, 3, 3))
    idx = [(0, 0, 0), (0, 1, 1), (0, 2, 2), (1, 1, 3), (1, 2, 4), (2, 2, 5)]
    for a, b, c in idx:
        Cs_m[:, a, b] = Cs[:, c]
        Cs_m[:, b, a] = Cs[:, c]
    Cs_l = np.einsum("ji,njk,kl->nil", R, Cs_m, R)
    Cs_local = np.stack([Cs_l[:, a, b] for a, b, _ in idx], 1)
    mu = np.concatenate([ps_local, pt]).astype(np.float32)
    cov = np.concatenate([Cs_local, Ct]).astype(np.float32)
    nrm = np.concatenate([ns_local, nt]).astype(np.float32)
    gt = np.stack([T_s, _pose(np.eye(3), np.zeros(3))])
    poses = gt.copy()
    poses[0] = perturb_poses(gt[:1], seed + 100)[0]
    return Scene("C1", mu, cov, nrm, np.array([0, n, 2 * n], np.int64), np.array([1], np.int64),
                 1.0, 1, np.array([[0, 0, 0, 1, 1]], np.int64), poses, gt,
                 np.array([[0, 0, 0, 1]], np.int64), 0)


def odometry_step(seed=2, n_kf=10, kf_spacing=2.0, n_points=20000, rings=128, az=1024):
    """C2: newest 20k-point frame vs 10 keyframe maps spaced ~2 m, r = 0.25/0.5/1.0."""
    path = StreetPath(seed, 400.0, 5)
    world = _World(5)
    s0 = 25.0 + n_kf * kf_spacing
    ss = [s0] + [s0 - kf_spacing * (k + 1) for k in range(n_kf)]
    gt = np.stack([path.pose(s, tilt_id=int(round(s * 100))) for s in ss])
    mu, cov, nrm, off = _make_clouds(world.h, gt, gt, 1, rings, az, 0.25, n_points, seed, 0)
    factors = np.array([[0, k, 0, k + 1, 1] for k in range(n_kf)], np.int64)
    pairs = np.array([[0, k, 0, k + 1] for k in range(n_kf)], np.int64)
    return Scene("C2", mu, cov, nrm, off, np.arange(1, n_kf + 1, dtype=np.int64), 0.25, 3,
                 factors, perturb_poses(gt, seed + 100), gt, pairs, 2)


def smoother_window(seed=3, n_frames=30, n_kf=20, per_frame=10, n_points=20000, rings=128,
                    az=1024):
    """C3: 30 consecutive frames x 10 of 20 keyframe factors each, 20k points, one batch."""
    path = StreetPath(seed, 400.0, 5)
    world = _World(5)
    s0 = 20.0 + 2.0 * n_kf
    ss_f = [s0 + 0.15 * f for f in range(n_frames)]           # 10 Hz at 1.5 m/s
    ss_k = [s0 - 2.0 * (k + 1) for k in range(n_kf)]
    ss = ss_f + ss_k
    gt = np.stack([path.pose(s, tilt_id=int(round(s * 100))) for s in ss])
    mu, cov, nrm, off = _make_clouds(world.h, gt, gt, 1, rings, az, 0.25, n_points, seed, 0)
    rs = np.random.default_rng(seed + 7)
    fl = []
    for f in range(n_frames):
        for k in sorted(rs.choice(n_kf, per_frame, replace=False)):
            fl.append([f, k, f, n_frames + k, 1])
    factors = np.array(fl, np.int64)
    pairs = factors[:, :4].copy()
    return Scene("C3", mu, cov, nrm, off, np.arange(n_frames, n_frames + n_kf, dtype=np.int64),
                 0.25, 3, factors, perturb_poses(gt, seed + 100), gt, pairs, 2)


def submap_scene(name, seed, n_submaps, n_points, half_blocks, factor_dist, cand_dist,
                 spacing=3.0, frames_per_submap=15, rings=128, az=1024, ds_res=0.1,
                 order_random=False, threads=None):
    """C4/C5: submaps (15 frames merged in the centre-frame origin) every 3 m
    along a street random walk; factors = pairs (newer source, older target) with
    origin distance < factor_dist; overlap candidates = pairs within cand_dist
    (stand-in for an AABB prefilter).  Both distances are taken between the
    LINEARIZATION poses (the perturbed estimates a mapping system holds), not
    the ground truth.  Submap frames use the sensor's full 1024 azimuth steps
    (SURVEY 8(d)), enough returns for exactly n_points per submap after the
    0.1 m downsampling.  r = 0.5/1.0/2.0 m (Q14)."""
    path = StreetPath(seed, n_submaps * spacing + 10.0, half_blocks)
    world = _World(half_blocks)
    s_c = np.array([5.0 + spacing * i for i in range(n_submaps)])
    origins = np.stack([path.pose(s, tilt_id=int(round(s * 100))) for s in s_c])
    frames = []
    for i in range(n_submaps):
        for f in range(frames_per_submap):
            s = s_c[i] + (f - frames_per_submap // 2) * (spacing / frames_per_submap)
            if f == frames_per_submap // 2:
                frames.append(origins[i])
            else:
                frames.append(path.pose(s, tilt_id=int(round(s * 100)) + 7))
    frames = np.stack(frames)
    mu, cov, nrm, off = _make_clouds(world.h, frames, origins, frames_per_submap, rings, az,
                                     ds_res, n_points, seed, 0, order_random, threads)
    lin = perturb_poses(origins, seed + 100)
    pos = lin.reshape(-1, 3, 4)[:, :, 3]
    fl, pl = [], []
    for i in range(n_submaps):
        d = np.linalg.norm(pos[:i] - pos[i], axis=1)
        for j in np.nonzero(d < cand_dist)[0]:
            pl.append([i, j, i, j])
            if d[j] < factor_dist:
                fl.append([i, j, i, j, 0])
    factors = np.array(fl, np.int64).reshape(-1, 5)
    pairs = np.array(pl, np.int64).reshape(-1, 4)
    return Scene(name, mu, cov, nrm, off, np.arange(n_submaps, dtype=np.int64), 0.5, 3, factors,
                 lin, origins, pairs, 1)


def global_scene(seed=4, **kw):
    """C4: 500 submaps x 50k points, ~1e4 factors."""
    args = dict(n_submaps=500, n_points=50000, half_blocks=5, factor_dist=60.0, cand_dist=90.0)
    args.update(kw)
    return submap_scene("C4", seed, **args)


def large_map_scene(seed=5, **kw):
    """C5: 2000 submaps x 100k points, ~1e5 factors + overlap screening."""
    args = dict(n_submaps=2000, n_points=100000, half_blocks=13, factor_dist=60.0,
                cand_dist=90.0)
    args.update(kw)
    return submap_scene("C5", seed, **args)


CONFIGS = {"C1": room_corner, "C2": odometry_step, "C3": smoother_window, "C4": global_scene,
           "C5": large_map_scene}


def make(name: str, **kw) -> Scene:
    return CONFIGS[name](**kw)
