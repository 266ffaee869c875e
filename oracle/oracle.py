"""ctypes front end of the fp64 CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2407_10344_b200) never imports this module.

Everything here is argument marshalling; the arithmetic lives in oracle.cpp,
which cites the paper passage each step follows (Sec. III-C,
Eqs. 2-8; overlap P:280).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

MAX_LEVELS = 8


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++ -O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared",
               "-fPIC", "-pthread", _SRC, "-o", _LIB + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class OracleFactor(ctypes.Structure):
    _fields_ = [
        ("H", ctypes.c_double * 144),
        ("b", ctypes.c_double * 12),
        ("e", ctypes.c_double),
        ("H_abs", ctypes.c_double * 144),
        ("b_abs", ctypes.c_double * 12),
        ("inliers", ctypes.c_int32 * MAX_LEVELS),
        ("num_invisible", ctypes.c_int64),
        ("num_degenerate", ctypes.c_int64),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.oracle_build_voxelmap.restype = P
        L.oracle_build_voxelmap.argtypes = [P, P, ctypes.c_int64, ctypes.c_double, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_int)]
        L.oracle_map_free.argtypes = [P]
        L.oracle_map_num_voxels.restype = ctypes.c_int64
        L.oracle_map_num_voxels.argtypes = [P, ctypes.c_int]
        L.oracle_map_export.argtypes = [P, ctypes.c_int, P, P, P, P]
        L.oracle_lookup.restype = ctypes.c_int64
        L.oracle_lookup.argtypes = [P, ctypes.c_int, P]
        L.oracle_pack_key.restype = ctypes.c_int64
        L.oracle_pack_key.argtypes = [ctypes.c_int64] * 3
        L.oracle_relative_pose.argtypes = [P, P, P, P]
        L.oracle_overlap.restype = ctypes.c_int64
        L.oracle_overlap.argtypes = [P, ctypes.c_int64, P, P, P, ctypes.c_int]
        L.oracle_linearize.argtypes = [P, P, P, ctypes.c_int64, P, P, P, ctypes.c_int, P, P, P, P]
        L.oracle_linearize_batch.argtypes = [P, P, P, P, P, P, ctypes.c_int64, P, ctypes.c_int, P]
        L.oracle_overlap_batch.argtypes = [P, P, P, P, ctypes.c_int64, P, ctypes.c_int,
                                           ctypes.c_int, P]
        L.oracle_overlap_union.restype = ctypes.c_int64
        L.oracle_overlap_union.argtypes = [P, ctypes.c_int64, P, P, ctypes.c_int64, P, ctypes.c_int]
        L.oracle_sizeof_factor.restype = ctypes.c_int
        assert L.oracle_sizeof_factor() == ctypes.sizeof(OracleFactor)
        _lib = L
    return _lib


def _f32(a, cols):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1, cols))
    return a


def _f64(a, n):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
    assert a.size == n, a.shape
    return a


def _ptr(a):
    return None if a is None else a.ctypes.data


class VoxelMap:
    """Oracle multi-resolution voxelmap.  Level l has r_l = r0 * 2**l."""

    def __init__(self, mu, cov, r0: float, levels: int):
        self.mu = _f32(mu, 3)
        self.cov = _f32(cov, 6)
        assert self.mu.shape[0] == self.cov.shape[0]
        st = ctypes.c_int(0)
        h = lib().oracle_build_voxelmap(_ptr(self.mu), _ptr(self.cov), self.mu.shape[0],
                                        float(r0), int(levels), ctypes.byref(st))
        if not h:
            raise ValueError("oracle_build_voxelmap failed: " +
                             ("voxel key out of range" if st.value == 1 else "invalid arguments"))
        self.handle = ctypes.c_void_p(h)
        self.r0 = float(r0)
        self.levels = int(levels)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.oracle_map_free(h)
            self.handle = None

    def num_voxels(self, level: int) -> int:
        return int(lib().oracle_map_num_voxels(self.handle, level))

    def export(self, level: int):
        """(keys int64 [V], means f64 [V,3], covs f64 [V,6], counts int64 [V]), ascending key."""
        V = self.num_voxels(level)
        keys = np.empty(V, np.int64)
        means = np.empty((V, 3), np.float64)
        covs = np.empty((V, 6), np.float64)
        counts = np.empty(V, np.int64)
        lib().oracle_map_export(self.handle, level, _ptr(keys), _ptr(means), _ptr(covs),
                                _ptr(counts))
        return keys, means, covs, counts

    def lookup(self, level: int, q) -> int:
        q = _f64(q, 3)
        return int(lib().oracle_lookup(self.handle, level, _ptr(q)))


def pack_key(kx: int, ky: int, kz: int) -> int:
    return int(lib().oracle_pack_key(int(kx), int(ky), int(kz)))


def relative_pose(Ti, Tj):
    """T_ij = T_j^-1 T_i (3x4) and viewpoint v = T_i^-1 t_j (reading Q1/R1)."""
    Ti = _f64(Ti, 12)
    Tj = _f64(Tj, 12)
    out = np.empty(12, np.float64)
    v = np.empty(3, np.float64)
    lib().oracle_relative_pose(_ptr(Ti), _ptr(Tj), _ptr(out), _ptr(v))
    return out.reshape(3, 4), v


def overlap(mu, vmap: VoxelMap, Ti, Tj, level: int) -> int:
    mu = _f32(mu, 3)
    Ti = _f64(Ti, 12)
    Tj = _f64(Tj, 12)
    return int(lib().oracle_overlap(_ptr(mu), mu.shape[0], vmap.handle, _ptr(Ti), _ptr(Tj),
                                    int(level)))


def overlap_union(mu, vmaps, Ti, Tjs, level: int) -> int:
    """Points of mu (at Ti) falling in a voxel of ANY of vmaps (map k at Tjs[k])."""
    mu = _f32(mu, 3)
    Ti = _f64(Ti, 12)
    K = len(vmaps)
    Tjs = _f64(np.asarray(Tjs, np.float64).reshape(-1), 12 * K)
    P = ctypes.c_void_p
    mh = (P * max(K, 1))(*[m.handle.value for m in vmaps])
    return int(lib().oracle_overlap_union(_ptr(mu), mu.shape[0], mh, _ptr(Tjs), K, _ptr(Ti),
                                          int(level)))


def _factor_dict(f: OracleFactor, levels: int):
    H = np.ctypeslib.as_array(f.H).reshape(12, 12).copy()
    b = np.ctypeslib.as_array(f.b).copy()
    return {
        "H": H, "b": b, "e": float(f.e),
        "H_abs": np.ctypeslib.as_array(f.H_abs).reshape(12, 12).copy(),
        "b_abs": np.ctypeslib.as_array(f.b_abs).copy(),
        "H_ii": H[:6, :6], "H_ij": H[:6, 6:], "H_jj": H[6:, 6:],
        "b_i": b[:6], "b_j": b[6:],
        "inliers": np.array(f.inliers[:levels], np.int64),
        "num_invisible": int(f.num_invisible),
        "num_degenerate": int(f.num_degenerate),
    }


def linearize(mu, cov, normals, vmap: VoxelMap, Ti, Tj, validate: bool = False,
              eval_Ti=None, eval_Tj=None, return_corr: bool = False):
    """One matching cost factor (Eqs. 2-8).  Returns a dict of fp64 results."""
    mu = _f32(mu, 3)
    cov = _f32(cov, 6)
    nrm = None if normals is None else _f32(normals, 3)
    n = mu.shape[0]
    Ti = _f64(Ti, 12)
    Tj = _f64(Tj, 12)
    eTi = None if eval_Ti is None else _f64(eval_Ti, 12)
    eTj = None if eval_Tj is None else _f64(eval_Tj, 12)
    out = OracleFactor()
    corr = np.empty((n, vmap.levels), np.int64) if return_corr else None
    lib().oracle_linearize(_ptr(mu), _ptr(cov), _ptr(nrm), n, vmap.handle, _ptr(Ti), _ptr(Tj),
                           int(bool(validate)), _ptr(eTi), _ptr(eTj), ctypes.byref(out),
                           _ptr(corr))
    d = _factor_dict(out, vmap.levels)
    if return_corr:
        d["corr"] = corr
    return d


def linearize_batch(clouds, maps, factors, poses, num_threads: int = 1):
    """clouds: list of (mu, cov, normals|None); maps: list of VoxelMap;
    factors: int64 [F,5] {source, target, pose_i, pose_j, flags}; poses [P,12]."""
    clouds = [(_f32(m, 3), _f32(c, 6), None if n is None else _f32(n, 3)) for m, c, n in clouds]
    factors = np.ascontiguousarray(np.asarray(factors, np.int64).reshape(-1, 5))
    poses = np.ascontiguousarray(np.asarray(poses, np.float64).reshape(-1, 12))
    F = factors.shape[0]
    P = ctypes.c_void_p
    mus = (P * len(clouds))(*[c[0].ctypes.data for c in clouds])
    covs = (P * len(clouds))(*[c[1].ctypes.data for c in clouds])
    nrms = (P * len(clouds))(*[(c[2].ctypes.data if c[2] is not None else None) for c in clouds])
    npts = np.array([c[0].shape[0] for c in clouds], np.int64)
    mh = (P * len(maps))(*[m.handle.value for m in maps])
    out = (OracleFactor * max(F, 1))()
    lib().oracle_linearize_batch(mus, covs, nrms, _ptr(npts), mh, _ptr(factors), F, _ptr(poses),
                                 int(num_threads), out)
    levels = [maps[int(factors[f, 1])].levels for f in range(F)]
    return [_factor_dict(out[f], levels[f]) for f in range(F)]


def overlap_batch(mus, maps, pairs, poses, level: int, num_threads: int = 1):
    """pairs int64 [P,4] {source, target, pose_i, pose_j} -> counts int64 [P]."""
    mus = [_f32(m, 3) for m in mus]
    pairs = np.ascontiguousarray(np.asarray(pairs, np.int64).reshape(-1, 4))
    poses = np.ascontiguousarray(np.asarray(poses, np.float64).reshape(-1, 12))
    P = ctypes.c_void_p
    mp = (P * len(mus))(*[m.ctypes.data for m in mus])
    npts = np.array([m.shape[0] for m in mus], np.int64)
    mh = (P * len(maps))(*[m.handle.value for m in maps])
    counts = np.zeros(pairs.shape[0], np.int64)
    lib().oracle_overlap_batch(mp, _ptr(npts), mh, _ptr(pairs), pairs.shape[0], _ptr(poses),
                               int(level), int(num_threads), _ptr(counts))
    return counts
