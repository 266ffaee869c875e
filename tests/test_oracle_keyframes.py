"""Pins of the keyframe mechanism, CPU only.

* the removal rules on hand-worked overlap matrices (values computed by hand
  in the comments), for both the oracle (oracle/keyframes.py) and the
  library's host-only gvox_keyframe_update;
* the union overlap against brute-force membership of each point in
  each map (per-point lookups, themselves pinned by a brute-force scan in
  test_oracle_voxelmap.py), one map = the pair overlap, a repeated map counts
  once, disjoint maps add.
"""
import numpy as np
import pytest

from oracle import keyframes as okf

# 4 old keyframes + the latest (index 4); n_odom = 3, min_overlap = 0.05
O1 = np.array([
    [1.0, 0.6, 0.3, 0.2, 0.04],
    [0.5, 1.0, 0.7, 0.4, 0.30],
    [0.3, 0.6, 1.0, 0.8, 0.50],
    [0.2, 0.3, 0.7, 1.0, 0.60],
    [0.1, 0.3, 0.5, 0.6, 1.00]])
# rule 1: o(0, 4) = 0.04 < 0.05 -> remove 0.  Remaining {1, 2, 3, 4}: 4 > 3 ->
# s(1) = 0.30 * ((1 - 0.7) + (1 - 0.4)) = 0.27
# s(2) = 0.50 * ((1 - 0.6) + (1 - 0.8)) = 0.30
# s(3) = 0.60 * ((1 - 0.3) + (1 - 0.7)) = 0.60   -> remove 1.
R1 = [0, 1]
# same matrix, n_odom = 4: only rule 1 fires
R1b = [0]
# ties: three identical old keyframes, n_odom = 2 -> s equal, the first goes
O2 = np.array([[1, .5, .5, .5], [.5, 1, .5, .5], [.5, .5, 1, .5], [.5, .5, .5, 1.0]])
R2 = [0]


@pytest.mark.parametrize("o,n_odom,expect", [(O1, 3, R1), (O1, 4, R1b), (O2, 2, R2),
                                             (O2, 4, []), (np.ones((1, 1)), 1, [])])
def test_removal_rules_worked(o, n_odom, expect):
    assert okf.keyframe_update(o, n_odom, 0.05) == expect
    import paper_2407_10344_b200 as gv  # host-only entry point: no GPU needed
    assert np.flatnonzero(gv.keyframe_update(o, n_odom, 0.05)).tolist() == expect


def test_keyframe_update_errors():
    import paper_2407_10344_b200 as gv
    with pytest.raises(gv.GvoxError):
        gv.keyframe_update(np.full((2, 2), np.nan))
    with pytest.raises(gv.GvoxError):
        gv.keyframe_update(np.ones((2, 2)), n_odom=0)


def test_union_overlap_pins(oracle):
    rs = np.random.default_rng(7)
    pts = rs.uniform(-6, 6, (400, 3)).astype(np.float32)
    cov = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (400, 1))
    left, right = pts[pts[:, 0] < 0], pts[pts[:, 0] >= 0]
    mL = oracle.VoxelMap(left, cov[: len(left)], 0.5, 2)
    mR = oracle.VoxelMap(right, cov[: len(right)], 0.5, 2)
    I = np.eye(4)[:3].reshape(12)
    src = (pts + rs.normal(0, 0.3, pts.shape)).astype(np.float32)
    T = np.eye(4)
    T[:3, 3] = [0.2, -0.1, 0.05]
    Ti = T[:3].reshape(12)
    for level in (0, 1):
        # brute force: per point, membership in either map by lookup
        Tm = np.linalg.inv(np.eye(4)) @ T
        q = src.astype(float) @ Tm[:3, :3].T + Tm[:3, 3]
        hitL = np.array([mL.lookup(level, p) >= 0 for p in q])
        hitR = np.array([mR.lookup(level, p) >= 0 for p in q])
        u = oracle.overlap_union(src, [mL, mR], Ti, np.stack([I, I]), level)
        assert u == int((hitL | hitR).sum())
        # disjoint halves (x < 0 vs x >= 0 at voxel boundaries 0): counts add
        assert u == oracle.overlap(src, mL, Ti, I, level) + oracle.overlap(src, mR, Ti, I, level)
        assert oracle.overlap_union(src, [mL], Ti, I[None], level) == oracle.overlap(src, mL, Ti, I, level)
        assert oracle.overlap_union(src, [mL, mL], Ti, np.stack([I, I]), level) == \
            oracle.overlap(src, mL, Ti, I, level)
        assert oracle.overlap_union(src, [], Ti, np.zeros((0, 12)), level) == 0
