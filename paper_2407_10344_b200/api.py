"""Thin Python front end of libgvox (include/gvox.h).

Argument marshalling only: numpy arrays are host buffers, torch CUDA tensors are
device buffers (torch provides device memory and the CUDA stream), and every
computation runs in the library's sm_100a kernels.  Names follow the C ABI
(gvox_create_voxelmap -> create_voxelmap, gvox_overlap -> overlap,
gvox_linearize_batch -> linearize_batch, ...).
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from ._lib import (FACTOR_ACCUM_DTYPE, FACTOR_DTYPE, GVOX_DEVICE, GVOX_HOST, LINEAR_FACTOR_DTYPE,
                   PAIR_DTYPE, REGISTER_PARAMS_DTYPE, REGISTER_RESULT_DTYPE, UNION_MEMBER_DTYPE,
                   UNION_QUERY_DTYPE, GLOBAL_PARAMS_DTYPE, GLOBAL_RESULT_DTYPE,
                   OPTIMIZE_PARAMS_DTYPE, OPTIMIZE_RESULT_DTYPE, check, lib)


def _torch():
    import torch
    return torch


def _is_cuda_tensor(x) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def _ptr(x):
    """(pointer, mem) of a numpy array or torch CUDA tensor (contiguous)."""
    if x is None:
        return None, None
    if _is_cuda_tensor(x):
        assert x.is_contiguous(), "device tensors must be contiguous"
        return ctypes.c_void_p(x.data_ptr()), GVOX_DEVICE
    assert isinstance(x, np.ndarray) and x.flags["C_CONTIGUOUS"], type(x)
    return ctypes.c_void_p(x.ctypes.data), GVOX_HOST


def _out_ptr(ctx, out, n: int, dtype: np.dtype, what: str):
    """(pointer, mem) of an output buffer after checking it can hold n elements
    of `dtype`: a numpy array of that dtype, or a contiguous CUDA tensor on the
    context's device with at least n * itemsize bytes (record tensors: uint8
    [>= n, itemsize]).  An undersized or mistyped buffer raises instead of
    letting the library write past its end."""
    dtype = np.dtype(dtype)
    if _is_cuda_tensor(out):
        if out.device != ctx.device:
            raise ValueError(f"{what}: output on {out.device}, context on {ctx.device}")
        if not out.is_contiguous():
            raise ValueError(f"{what}: output tensor must be contiguous")
        if out.dim() == 2 and out.element_size() == 1 and out.shape[1] != dtype.itemsize:
            raise ValueError(f"{what}: record tensor rows are {out.shape[1]} B, need {dtype.itemsize}")
        if out.dim() != 2 and out.element_size() != dtype.itemsize:
            raise ValueError(f"{what}: output element size {out.element_size()}, need {dtype.itemsize}")
        if out.numel() * out.element_size() < n * dtype.itemsize:
            raise ValueError(f"{what}: output holds {out.numel() * out.element_size()} B, "
                             f"need {n} x {dtype.itemsize} B")
        return ctypes.c_void_p(out.data_ptr()), GVOX_DEVICE
    if not isinstance(out, np.ndarray) or not out.flags["C_CONTIGUOUS"]:
        raise ValueError(f"{what}: output must be a contiguous numpy array or CUDA tensor")
    if out.dtype != dtype or out.size < n:
        raise ValueError(f"{what}: output {out.dtype} [{out.size}], need {dtype} [>= {n}]")
    return ctypes.c_void_p(out.ctypes.data), GVOX_HOST


class Context:
    """gvox_ctx on one CUDA device, enqueuing on a torch stream (default: the
    device's current stream)."""

    def __init__(self, device: int = 0, stream=None):
        torch = _torch()
        self.device_index = int(device)
        self.device = torch.device("cuda", self.device_index)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        h = ctypes.c_void_p()
        check(lib().gvox_ctx_create(self.device_index, ctypes.c_void_p(stream.cuda_stream),
                                    ctypes.byref(h)))
        self.handle = h

    def enable_timing(self, enable: bool = True):
        """Bracket the library's kernel launches with CUDA events (gvox_ctx_enable_timing)."""
        check(lib().gvox_ctx_enable_timing(self.handle, int(bool(enable))))

    def timing(self, reset: bool = False) -> dict:
        """{group: (ms, launches)} for groups build/overlap/linearize/reduce (synchronizes)."""
        from ._lib import TIMERS
        ms = (ctypes.c_double * len(TIMERS))()
        n = (ctypes.c_int64 * len(TIMERS))()
        check(lib().gvox_ctx_timing(self.handle, ms, n, int(bool(reset))))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(TIMERS)}

    def set_stream(self, stream):
        self.stream = stream
        check(lib().gvox_ctx_set_stream(self.handle, ctypes.c_void_p(stream.cuda_stream)))

    def close(self):
        if getattr(self, "handle", None):
            lib().gvox_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass


class Cloud:
    """gvox_cloud: Gaussian points copied into device-resident planar float4
    arrays.  mu [n,3], cov [n,6] (xx xy xz yy yz zz), normals [n,3] or None;
    numpy (host) or torch CUDA tensors (device), float32."""

    def __init__(self, ctx: Context, mu, cov, normals=None, *, _handle=None, _n=None):
        if _handle is not None:
            self.handle = _handle
            self.n = int(_n)
            return
        if not _is_cuda_tensor(mu):
            mu = np.ascontiguousarray(np.asarray(mu, np.float32).reshape(-1, 3))
            cov = np.ascontiguousarray(np.asarray(cov, np.float32).reshape(-1, 6))
            if normals is not None:
                normals = np.ascontiguousarray(np.asarray(normals, np.float32).reshape(-1, 3))
        n = int(mu.shape[0])
        pm, mem = _ptr(mu)
        pc, _ = _ptr(cov)
        pn, _ = _ptr(normals)
        h = ctypes.c_void_p()
        check(lib().gvox_cloud_create(ctx.handle, pm, pc, pn, n, mem, ctypes.byref(h)))
        self.handle = h
        self.n = n

    def __len__(self):
        return self.n

    def close(self):
        if getattr(self, "handle", None):
            lib().gvox_cloud_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass


def create_clouds(ctx: Context, mu, cov, normals, offsets):
    """gvox_clouds_create: many clouds stored back to back (cloud k = rows
    offsets[k]:offsets[k+1]); numpy (host, ideally pinned) or CUDA tensors."""
    offsets = np.ascontiguousarray(np.asarray(offsets, np.int64))
    count = len(offsets) - 1
    if not _is_cuda_tensor(mu):
        mu = np.ascontiguousarray(np.asarray(mu, np.float32).reshape(-1, 3))
        cov = np.ascontiguousarray(np.asarray(cov, np.float32).reshape(-1, 6))
        if normals is not None:
            normals = np.ascontiguousarray(np.asarray(normals, np.float32).reshape(-1, 3))
    pm, mem = _ptr(mu)
    out = (ctypes.c_void_p * max(count, 1))()
    check(lib().gvox_clouds_create(ctx.handle, pm, _ptr(cov)[0], _ptr(normals)[0],
                                   _ptr(offsets)[0], count, mem, out))
    return [Cloud(ctx, None, None, _handle=ctypes.c_void_p(out[k]),
                  _n=int(offsets[k + 1] - offsets[k])) for k in range(count)]


class VoxelMap:
    """gvox_map: multi-resolution Gaussian voxelmap."""

    def __init__(self, handle: ctypes.c_void_p, levels: int = None, batch=None):
        self.handle = handle
        self.levels = int(lib().gvox_voxelmap_levels(handle)) if levels is None else int(levels)
        self._batch = batch  # _MapBatch of create_voxelmaps: destroys the maps left in one call

    def info(self, level: int):
        n = ctypes.c_int64()
        r = ctypes.c_double()
        check(lib().gvox_voxelmap_info(self.handle, level, ctypes.byref(n), ctypes.byref(r)))
        return int(n.value), float(r.value)

    def num_voxels(self, level: int) -> int:
        return self.info(level)[0]

    def export(self, ctx: Context, level: int):
        """(keys int64 [V], means f64 [V,3], covs f64 [V,6], counts int32 [V]) in
        ascending packed-key order."""
        V = self.num_voxels(level)
        keys = np.empty(V, np.int64)
        means = np.empty((V, 3), np.float64)
        covs = np.empty((V, 6), np.float64)
        counts = np.empty(V, np.int32)
        check(lib().gvox_voxelmap_export(ctx.handle, self.handle, level, _ptr(keys)[0],
                                         _ptr(means)[0], _ptr(covs)[0], _ptr(counts)[0]))
        return keys, means, covs, counts

    def lookup(self, ctx: Context, level: int, q):
        """Packed key of the voxel containing each q (fp64 [n,3]) or -1."""
        if _is_cuda_tensor(q):
            torch = _torch()
            out = torch.empty(q.shape[0], dtype=torch.int64, device=q.device)
        else:
            q = np.ascontiguousarray(np.asarray(q, np.float64).reshape(-1, 3))
            out = np.empty(q.shape[0], np.int64)
        pq, mem = _ptr(q)
        check(lib().gvox_voxelmap_lookup(ctx.handle, self.handle, level, pq, int(q.shape[0]),
                                         _ptr(out)[0], mem))
        return out

    def close(self):
        if getattr(self, "handle", None):
            if self._batch is not None:
                self._batch.release(self.handle)
            lib().gvox_map_destroy(self.handle)
            self.handle = None

    def __del__(self):
        # a batch member is destroyed with its batch (one call for all of them)
        if getattr(self, "_batch", None) is not None:
            return
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass


class _MapBatch:
    """The maps of one create_voxelmaps call: whatever its VoxelMaps have not
    closed explicitly is destroyed with ONE gvox_maps_destroy call when the
    last of them goes (each VoxelMap holds a reference)."""

    def __init__(self, handles):
        self.arr = handles  # ctypes array of gvox_map*
        self.n = len(handles)

    def release(self, handle):
        for i in range(self.n):
            if self.arr[i] == handle.value:
                self.arr[i] = None

    def __del__(self):
        try:
            lib().gvox_maps_destroy(self.arr, self.n)
        except Exception:  # pragma: no cover
            pass


def create_voxelmap(ctx: Context, cloud: Cloud, r0: float, levels: int) -> VoxelMap:
    h = ctypes.c_void_p()
    check(lib().gvox_create_voxelmap(ctx.handle, cloud.handle, float(r0), int(levels),
                                     ctypes.byref(h)))
    return VoxelMap(h)


def create_voxelmaps(ctx: Context, clouds: Sequence[Cloud], r0: float, levels: int):
    n = len(clouds)
    arr = (ctypes.c_void_p * max(n, 1))(*[c.handle.value for c in clouds])
    out = (ctypes.c_void_p * max(n, 1))()
    check(lib().gvox_create_voxelmaps(ctx.handle, arr, n, float(r0), int(levels), out))
    batch = _MapBatch(out)
    return [VoxelMap(ctypes.c_void_p(out[i]), levels, batch) for i in range(n)]


class HandleArray:
    """Pre-built array of handles (avoids rebuilding it on every call)."""

    def __init__(self, objs):
        self.objs = list(objs)
        self.n = len(self.objs)
        self.arr = (ctypes.c_void_p * max(self.n, 1))(*[o.handle.value for o in self.objs])


def _handles(objs):
    return objs if isinstance(objs, HandleArray) else HandleArray(objs)


def as_factors(factors) -> np.ndarray:
    f = np.asarray(factors)
    if f.dtype == FACTOR_DTYPE:
        return np.ascontiguousarray(f)
    f = f.reshape(-1, 5).astype(np.int64)
    out = np.empty(f.shape[0], FACTOR_DTYPE)
    for i, name in enumerate(FACTOR_DTYPE.names):
        out[name] = f[:, i]
    return out


def as_pairs(pairs) -> np.ndarray:
    p = np.asarray(pairs)
    if p.dtype == PAIR_DTYPE:
        return np.ascontiguousarray(p)
    p = p.reshape(-1, 4).astype(np.int64)
    out = np.empty(p.shape[0], PAIR_DTYPE)
    for i, name in enumerate(PAIR_DTYPE.names):
        out[name] = p[:, i]
    return out


def as_poses(poses) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(poses, np.float64).reshape(-1, 12))


def overlap(ctx: Context, clouds, maps, pairs, poses, level: int, out=None):
    """gvox_overlap: int32 counts per pair (numpy, or into the int32 CUDA tensor `out`)."""
    C, M = _handles(clouds), _handles(maps)
    pairs = as_pairs(pairs)
    poses = as_poses(poses)
    if out is None:
        out = np.empty(pairs.shape[0], np.int32)
    po, mem = _out_ptr(ctx, out, pairs.shape[0], np.int32, "overlap")
    check(lib().gvox_overlap(ctx.handle, C.arr, C.n, M.arr, M.n, _ptr(pairs)[0], pairs.shape[0],
                             _ptr(poses)[0], poses.shape[0], int(level), po, mem))
    return out


def overlap_select(ctx: Context, clouds, maps, pairs, poses, level: int, num: int = 1,
                   den: int = 20, out=None):
    """gvox_overlap_select: uint8 decisions count * den > n * num per pair (default:
    overlap rate exceeds 5 %), exact, with early termination per pair."""
    C, M = _handles(clouds), _handles(maps)
    pairs = as_pairs(pairs)
    poses = as_poses(poses)
    if out is None:
        out = np.empty(pairs.shape[0], np.uint8)
    po, mem = _out_ptr(ctx, out, pairs.shape[0], np.uint8, "overlap_select")
    check(lib().gvox_overlap_select(ctx.handle, C.arr, C.n, M.arr, M.n, _ptr(pairs)[0],
                                    pairs.shape[0], _ptr(poses)[0], poses.shape[0], int(level),
                                    int(num), int(den), po, mem))
    return out


def device_records(ctx: Context, n: int, dtype: np.dtype):
    torch = _torch()
    return torch.empty((n, dtype.itemsize), dtype=torch.uint8, device=ctx.device)


def records_to_numpy(t, dtype: np.dtype = LINEAR_FACTOR_DTYPE) -> np.ndarray:
    if _is_cuda_tensor(t):
        t = t.cpu().numpy()
    return np.ascontiguousarray(t).view(dtype).reshape(-1)


def linearize_batch(ctx: Context, clouds, maps, factors, poses, out=None, corr_dump=None):
    """gvox_linearize_batch.  Returns a numpy structured array of
    LINEAR_FACTOR_DTYPE (host) or fills the uint8 CUDA tensor `out`
    ([F, 1008], see device_records).  corr_dump: optional int64 CUDA tensor
    [sum_f N_f * L_f]."""
    C, M = _handles(clouds), _handles(maps)
    factors = as_factors(factors)
    poses = as_poses(poses)
    F = factors.shape[0]
    if out is None:
        out = np.zeros(F, LINEAR_FACTOR_DTYPE)
    po, mem = _out_ptr(ctx, out, F, LINEAR_FACTOR_DTYPE, "linearize_batch")
    pc = None
    if corr_dump is not None:
        if not _is_cuda_tensor(corr_dump):
            raise ValueError("linearize_batch: corr_dump must be an int64 CUDA tensor")
        pc, _ = _out_ptr(ctx, corr_dump, corr_dump_size(C.objs, M.objs, factors), np.int64,
                         "linearize_batch corr_dump")
    check(lib().gvox_linearize_batch(ctx.handle, C.arr, C.n, M.arr, M.n, _ptr(factors)[0], F,
                                     _ptr(poses)[0], poses.shape[0], po, mem, pc))
    return out


def linearize_batch_accum(ctx: Context, clouds, maps, factors, poses, out=None):
    """gvox_linearize_batch_accum: compact target-block records (FACTOR_ACCUM_DTYPE)."""
    C, M = _handles(clouds), _handles(maps)
    factors = as_factors(factors)
    poses = as_poses(poses)
    F = factors.shape[0]
    if out is None:
        out = np.zeros(F, FACTOR_ACCUM_DTYPE)
    po, mem = _out_ptr(ctx, out, F, FACTOR_ACCUM_DTYPE, "linearize_batch_accum")
    check(lib().gvox_linearize_batch_accum(ctx.handle, C.arr, C.n, M.arr, M.n, _ptr(factors)[0], F,
                                           _ptr(poses)[0], poses.shape[0], po, mem))
    return out


def linearize_batch_accum_select(ctx: Context, clouds, maps, candidates, selected, poses, out,
                                 selected_host=None):
    """gvox_linearize_batch_accum_select: linearize the candidates whose device
    decision `selected` (uint8 CUDA tensor, e.g. overlap_select(..., out=<CUDA
    tensor>)) is set, compacted on the device in candidate order, into the
    uint8 CUDA tensor `out` ([>= len(candidates), 288]).  Returns the number
    selected; `selected_host` (optional uint8 numpy array) receives the
    decisions."""
    C, M = _handles(clouds), _handles(maps)
    candidates = as_factors(candidates)
    poses = as_poses(poses)
    F = candidates.shape[0]
    if not (_is_cuda_tensor(selected) and _is_cuda_tensor(out)):
        raise ValueError("linearize_batch_accum_select: selected and out must be CUDA tensors")
    _out_ptr(ctx, selected, F, np.uint8, "linearize_batch_accum_select selected")
    _out_ptr(ctx, out, F, FACTOR_ACCUM_DTYPE, "linearize_batch_accum_select")
    ns = ctypes.c_int64(0)
    sh = None
    if selected_host is not None:
        assert selected_host.dtype == np.uint8 and selected_host.shape[0] >= F
        sh = _ptr(selected_host)[0]
    check(lib().gvox_linearize_batch_accum_select(
        ctx.handle, C.arr, C.n, M.arr, M.n, _ptr(candidates)[0], F,
        ctypes.c_void_p(selected.data_ptr()), _ptr(poses)[0], poses.shape[0],
        ctypes.c_void_p(out.data_ptr()), ctypes.byref(ns), sh))
    return int(ns.value)


def expand(ctx: Context, factors, poses, accum, out=None):
    """gvox_expand: compact records (uint8 CUDA tensor [F, 288]) -> full records."""
    factors = as_factors(factors)
    poses = as_poses(poses)
    F = factors.shape[0]
    if not _is_cuda_tensor(accum):
        raise ValueError("expand: accum must be a CUDA tensor")
    _out_ptr(ctx, accum, F, FACTOR_ACCUM_DTYPE, "expand accum")
    if out is None:
        out = np.zeros(F, LINEAR_FACTOR_DTYPE)
    po, mem = _out_ptr(ctx, out, F, LINEAR_FACTOR_DTYPE, "expand")
    check(lib().gvox_expand(ctx.handle, _ptr(factors)[0], F, _ptr(poses)[0], poses.shape[0],
                            ctypes.c_void_p(accum.data_ptr()), po, mem))
    return out


def _points_batch(points, offsets):
    if _is_cuda_tensor(points):
        pts = points.to(_torch().float32).reshape(-1, 3).contiguous()
    else:
        pts = np.ascontiguousarray(np.asarray(points, np.float32).reshape(-1, 3))
    n = pts.shape[0]
    off = np.array([0, n] if offsets is None else offsets, np.int64)
    return pts, off


def knn(ctx: Context, points, k: int = 10, cell_size: float = 0.5, offsets=None):
    """gvox_knn: exact k nearest neighbours (local indices, -1 pad) of each
    point within its cloud.  points: float32 [N,3] numpy (-> numpy result) or
    CUDA tensor (-> int32 CUDA tensor); offsets: cloud boundaries [C+1]
    (default: one cloud)."""
    pts, off = _points_batch(points, offsets)
    n = pts.shape[0]
    if _is_cuda_tensor(pts):
        out = _torch().empty((n, k), dtype=_torch().int32, device=pts.device)
    else:
        out = np.empty((n, k), np.int32)
    pp_, mem = _ptr(pts)
    check(lib().gvox_knn(ctx.handle, pp_, _ptr(off)[0], len(off) - 1, int(k), float(cell_size),
                         _ptr(out)[0], mem))
    return out


def estimate_covariances(ctx: Context, points, neighbors, offsets=None):
    """gvox_estimate_covariances: (cov [N,6] fp32, normals [N,3] fp32), numpy
    or CUDA tensors like the inputs."""
    pts, off = _points_batch(points, offsets)
    n = pts.shape[0]
    k = int(neighbors.shape[1])
    if _is_cuda_tensor(pts):
        torch = _torch()
        nb = neighbors.to(torch.int32).contiguous()
        cov = torch.empty((n, 6), dtype=torch.float32, device=pts.device)
        nrm = torch.empty((n, 3), dtype=torch.float32, device=pts.device)
    else:
        nb = np.ascontiguousarray(np.asarray(neighbors, np.int32))
        cov = np.empty((n, 6), np.float32)
        nrm = np.empty((n, 3), np.float32)
    pp_, mem = _ptr(pts)
    check(lib().gvox_estimate_covariances(ctx.handle, pp_, _ptr(off)[0], len(off) - 1, _ptr(nb)[0],
                                          k, _ptr(cov)[0], _ptr(nrm)[0], mem))
    return cov, nrm


def overlap_union(ctx: Context, clouds, maps, queries, members, poses, level: int, out=None):
    """gvox_overlap_union: queries [Q,4] {source_cloud, pose_i, first, count},
    members [M,2] {target_map, pose_j}.  Returns int32 counts [Q] (host) or
    fills the int32 CUDA tensor `out`."""
    C, Mh = _handles(clouds), _handles(maps)
    q = np.ascontiguousarray(np.asarray(queries, np.int64).reshape(-1, 4).astype(np.int32)).view(
        UNION_QUERY_DTYPE).reshape(-1)
    m = np.ascontiguousarray(np.asarray(members, np.int64).reshape(-1, 2).astype(np.int32)).view(
        UNION_MEMBER_DTYPE).reshape(-1)
    poses = as_poses(poses)
    if out is None:
        out = np.zeros(len(q), np.int32)
    po, mem = _out_ptr(ctx, out, len(q), np.int32, "overlap_union")
    check(lib().gvox_overlap_union(ctx.handle, C.arr, C.n, Mh.arr, Mh.n, _ptr(q)[0], len(q),
                                   _ptr(m)[0] if len(m) else None, len(m), _ptr(poses)[0],
                                   poses.shape[0], int(level), po, mem))
    return out


def keyframe_update(overlap_rates, n_odom: int = 20, min_overlap: float = 0.05) -> np.ndarray:
    """gvox_keyframe_update (host): overlap_rates [K,K] o(i, j), row/col K-1 =
    the latest keyframe.  Returns a bool mask of the keyframes to remove."""
    o = np.ascontiguousarray(np.asarray(overlap_rates, np.float64))
    K = o.shape[0]
    rm = np.zeros(K, np.uint8)
    check(lib().gvox_keyframe_update(_ptr(o)[0], K, int(n_odom), float(min_overlap), _ptr(rm)[0]))
    return rm.astype(bool)


def keyframe_insert_test(count: int, n: int, num: int = 9, den: int = 10) -> bool:
    """gvox_keyframe_insert_test (host): P:280 insertion, den * count < num * n."""
    out = ctypes.c_int(0)
    check(lib().gvox_keyframe_insert_test(int(count), int(n), int(num), int(den), ctypes.byref(out)))
    return bool(out.value)


def keyframe_update_counts(counts, sizes, n_odom: int = 20, min_overlap: float = 0.05):
    """gvox_keyframe_update_counts (host): removal rules from raw overlap counts
    [K,K] and keyframe sizes [K].  Returns (remove mask, o(i, j) matrix)."""
    c = np.ascontiguousarray(np.asarray(counts, np.int64))
    n = np.ascontiguousarray(np.asarray(sizes, np.int64).reshape(-1))
    K = n.shape[0]
    assert c.shape == (K, K), (c.shape, K)
    rm = np.zeros(K, np.uint8)
    o = np.zeros((K, K), np.float64)
    check(lib().gvox_keyframe_update_counts(_ptr(c)[0], _ptr(n)[0], K, int(n_odom),
                                            float(min_overlap), _ptr(rm)[0], _ptr(o)[0]))
    return rm.astype(bool), o


class KeyframeList:
    """The P:280-288 keyframe mechanism driven through the library: for each
    new frame, one gvox_overlap_union and the insertion test
    gvox_keyframe_insert_test ("overlap with the union of all keyframes smaller
    than 90 %"), and on insertion one gvox_overlap of the new keyframe against
    the others (both directions) followed by gvox_keyframe_update_counts (the
    rates o(i, j) and the removal rules are formed in the library).  Holds only
    bookkeeping: the keyframes' frame ids, their raw pairwise overlap counts and
    point counts."""

    def __init__(self, ctx: Context, level: int, n_odom: int = 20, insert_num: int = 9,
                 insert_den: int = 10, min_overlap: float = 0.05):
        self.ctx, self.level, self.n_odom = ctx, int(level), int(n_odom)
        self.insert_num, self.insert_den, self.min_overlap = int(insert_num), int(insert_den), min_overlap
        self.frames = []          # frame ids of the keyframes, list order
        self.counts = np.zeros((0, 0), np.int64)   # counts[a, b]: points of a in b's voxels
        self.sizes = np.zeros(0, np.int64)
        self.o = np.zeros((0, 0))                  # the library's o(i, j) of the last update

    def add_frame(self, frame: int, clouds, maps, poses):
        """frame indexes clouds/maps/poses (its cloud, its voxelmap, its pose).
        Returns (inserted, removed frame ids)."""
        n = len(clouds[frame])
        if self.frames:
            members = [[f, f] for f in self.frames]
            cnt = int(overlap_union(self.ctx, clouds, maps, [[frame, frame, 0, len(members)]], members,
                                    poses, self.level)[0])
            if not keyframe_insert_test(cnt, n, self.insert_num, self.insert_den):
                return False, []
        ks = self.frames + [frame]
        K = len(ks)
        c = np.zeros((K, K), np.int64)
        c[:K - 1, :K - 1] = self.counts
        c[K - 1, K - 1] = n          # a cloud lies entirely in its own voxels
        sizes = np.append(self.sizes, n).astype(np.int64)
        if K > 1:
            pairs = [[f, frame, f, frame] for f in self.frames] + [[frame, f, frame, f] for f in self.frames]
            cc = overlap(self.ctx, clouds, maps, pairs, poses, self.level)
            c[:K - 1, K - 1] = cc[:K - 1]
            c[K - 1, :K - 1] = cc[K - 1:]
        rm, o = keyframe_update_counts(c, sizes, self.n_odom, self.min_overlap)
        keep = ~rm
        removed = [ks[a] for a in range(K) if rm[a]]
        self.frames = [ks[a] for a in range(K) if keep[a]]
        self.counts = c[np.ix_(keep, keep)]
        self.sizes = sizes[keep]
        self.o = o[np.ix_(keep, keep)]
        return True, removed


def solve_global(ctx: Context, factors, accum, poses, fixed, max_iterations: int = 500,
                 tol: float = 1e-10, lam: float = 0.0, dense: bool = False):
    """gvox_solve_global: one Gauss-Newton step of the whole factor graph.
    accum: compact records (numpy FACTOR_ACCUM_DTYPE, or a uint8 CUDA tensor
    [F, 288] -> delta is then a CUDA tensor).  Returns (delta [P,6], result,
    H [6V,6V] or None, b [6V] or None)."""
    factors = as_factors(factors)
    poses = as_poses(poses)
    NPz = poses.shape[0]
    fx = np.ascontiguousarray(np.asarray(fixed, np.uint8).reshape(-1))
    assert fx.size == NPz
    prm = np.zeros(1, GLOBAL_PARAMS_DTYPE)
    prm["max_iterations"], prm["tol"], prm["lambda"] = int(max_iterations), float(tol), float(lam)
    res = np.zeros(1, GLOBAL_RESULT_DTYPE)
    if _is_cuda_tensor(accum):
        delta = _torch().empty((NPz, 6), dtype=_torch().float64, device=accum.device)
        mem = GVOX_DEVICE
    else:
        accum = np.ascontiguousarray(accum)
        delta = np.zeros((NPz, 6), np.float64)
        mem = GVOX_HOST
    V = int(NPz - np.count_nonzero(fx))
    H = np.zeros((6 * V, 6 * V)) if dense else None
    b = np.zeros(6 * V) if dense else None
    check(lib().gvox_solve_global(ctx.handle, _ptr(factors)[0], factors.shape[0], _ptr(accum)[0],
                                  _ptr(poses)[0], NPz, _ptr(fx)[0], _ptr(prm)[0], _ptr(delta)[0],
                                  None if H is None else _ptr(H)[0], None if b is None else _ptr(b)[0],
                                  _ptr(res)[0], mem))
    return delta, res[0], H, b


def optimize_global(ctx: Context, clouds, maps, factors, poses, fixed, max_iterations: int = 10,
                    pcg_max_iterations: int = 2000, pcg_tol: float = 1e-10, lam: float = 0.0,
                    eps_rot: float = 1e-6, eps_trans: float = 1e-6):
    """gvox_optimize_global: Gauss-Newton over the whole graph on the device.
    Returns (poses_out [P,12], result, error_history [iterations])."""
    C, M = _handles(clouds), _handles(maps)
    factors = as_factors(factors)
    poses = as_poses(poses)
    NPz = poses.shape[0]
    fx = np.ascontiguousarray(np.asarray(fixed, np.uint8).reshape(-1))
    prm = np.zeros(1, OPTIMIZE_PARAMS_DTYPE)
    prm["max_iterations"], prm["pcg_max_iterations"] = int(max_iterations), int(pcg_max_iterations)
    prm["pcg_tol"], prm["lambda"] = float(pcg_tol), float(lam)
    prm["eps_rot"], prm["eps_trans"] = float(eps_rot), float(eps_trans)
    res = np.zeros(1, OPTIMIZE_RESULT_DTYPE)
    out = np.zeros((NPz, 12), np.float64)
    hist = np.zeros(max_iterations, np.float64)
    check(lib().gvox_optimize_global(ctx.handle, C.arr, C.n, M.arr, M.n, _ptr(factors)[0],
                                     factors.shape[0], _ptr(poses)[0], NPz, _ptr(fx)[0], _ptr(prm)[0],
                                     _ptr(out)[0], _ptr(hist)[0], _ptr(res)[0], GVOX_HOST))
    return out, res[0], hist[: int(res[0]["iterations"])]


def register_batch(ctx: Context, clouds, maps, factors, poses, max_iterations: int = 10,
                   lam: float = 0.0, eps_rot: float = 1e-6, eps_trans: float = 1e-6,
                   history: bool = False, device: bool = False):
    """gvox_register_batch: on-device Gauss-Newton over every factor's pose_i
    (variable) with pose_j fixed.  Returns (poses_out [P,12] f64, results
    [P] REGISTER_RESULT_DTYPE, history [max_iterations, P] f64 or None); with
    device=True the three are CUDA tensors (results as uint8 [P, 80])."""
    C, M = _handles(clouds), _handles(maps)
    factors = as_factors(factors)
    poses = as_poses(poses)
    NPz = poses.shape[0]
    prm = np.zeros(1, REGISTER_PARAMS_DTYPE)
    prm["max_iterations"], prm["lambda"] = int(max_iterations), float(lam)
    prm["eps_rot"], prm["eps_trans"] = float(eps_rot), float(eps_trans)
    if device:
        torch = _torch()
        dev = ctx.device
        pout = torch.empty((NPz, 12), dtype=torch.float64, device=dev)
        res = torch.empty((NPz, REGISTER_RESULT_DTYPE.itemsize), dtype=torch.uint8, device=dev)
        hist = torch.empty((max_iterations, NPz), dtype=torch.float64, device=dev) if history else None
        mem = GVOX_DEVICE
    else:
        pout = np.zeros((NPz, 12), np.float64)
        res = np.zeros(NPz, REGISTER_RESULT_DTYPE)
        hist = np.zeros((max_iterations, NPz), np.float64) if history else None
        mem = GVOX_HOST
    check(lib().gvox_register_batch(ctx.handle, C.arr, C.n, M.arr, M.n, _ptr(factors)[0],
                                    factors.shape[0], _ptr(poses)[0], NPz, _ptr(prm)[0],
                                    _ptr(pout)[0], _ptr(res)[0],
                                    None if hist is None else _ptr(hist)[0], mem))
    return pout, res, hist


def corr_dump_size(clouds: Sequence[Cloud], maps: Sequence[VoxelMap], factors) -> int:
    f = as_factors(factors)
    return int(sum(clouds[int(a)].n * maps[int(b)].levels
                   for a, b in zip(f["source_cloud"], f["target_map"])))


def full_blocks(rec) -> dict:
    """One LINEAR_FACTOR_DTYPE record -> dict of 6x6 / 6 numpy blocks."""
    return {"H_ii": rec["H_ii"].reshape(6, 6), "H_ij": rec["H_ij"].reshape(6, 6),
            "H_jj": rec["H_jj"].reshape(6, 6), "b_i": rec["b_i"], "b_j": rec["b_j"],
            "e": float(rec["error"]), "inliers": rec["inliers"].copy(),
            "num_invisible": int(rec["num_invisible"]),
            "num_degenerate": int(rec["num_degenerate"])}
