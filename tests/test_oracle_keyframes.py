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


# ---------------------------------------------------------------------------
# run_keyframes on a hand-worked sequence (P:280 insertion, P:282-283 removal).
# Frame f covers the unit cells x in SEQ_CELLS[f] (y = z = 0) of the world,
# one point per cell centre; it is stored in its own sensor frame under the
# pose POSE(f) (a multiple of 90 degrees of yaw and an integer translation,
# so every coordinate is exact).  With r = 1 the overlap o(a, b) is
# |cells_a & cells_b| / |cells_a| and the union overlap of a frame is
# |cells_f & (union of the keyframes' cells)| / |cells_f|.  n_odom = 3.
#
# f0  0..9   (10)  first frame: inserted.                         kf [0]
# f1  0..9   (10)  union 10/10 = 100 %: not inserted.             kf [0]
# f2  5..14  (10)  union 5/10: inserted; o(0,2) = 5/10.           kf [0, 2]
# f3  9..28  (20)  union {0..14}: 6/20: inserted; 3 <= n_odom.     kf [0, 2, 3]
# f4  14..33 (20)  union {0..28}: 15/20: inserted.  Rule 1: o(0,4) = 0 -> remove 0;
#                  o(2,4) = 1/10, o(3,4) = 15/20 stay; 3 remain.   kf [2, 3, 4]
# f5  16..35 (20)  union {5..33}: 18/20 = 90 % exactly: "smaller than 90 %" is
#                  false -> not inserted (10 * 18 < 9 * 20 is false).
# f6  10..39 (30)  union {5..33}: 24/30: inserted.  Rule 1: o(2,6) = 5/10,
#                  o(3,6) = 19/20, o(4,6) = 20/20 stay; 4 > 3 -> rule 2:
#                  s(2) = o(2,6)[(1 - o(2,3)) + (1 - o(2,4))] = .5 (.4 + .9)   = .65
#                  s(3) = o(3,6)[(1 - o(3,2)) + (1 - o(3,4))] = .95 (.7 + .25) = .9025
#                  s(4) = o(4,6)[(1 - o(4,2)) + (1 - o(4,3))] = 1 (.95 + .25)  = 1.2
#                  -> remove 2.                                    kf [3, 4, 6]
# f7  0..25  (26)  union {9..39}: 17/26: inserted.  o(3,7) = 17/20, o(4,7) = 12/20,
#                  o(6,7) = 16/30: no rule 1.  Rule 2 (4 > 3):
#                  s(3) = .85 [(1 - o(3,4)) + (1 - o(3,6))] = .85 (.25 + .05)  = .255
#                  s(4) = .6  [(1 - o(4,3)) + (1 - o(4,6))] = .6 (.25 + 0)     = .15
#                  s(6) = 16/30 [(1 - 19/30) + (1 - 20/30)] = 16/30 * 21/30    = .373
#                  -> remove 4.  (With o transposed, s'(i) = o(7,i) sum(1 - o(j,i)),
#                  the removal would differ.)                      kf [3, 6, 7]
# f8  28..41 (14)  union {0..39}: 12/14: inserted.  Rule 1: o(3,8) = 1/20 = 5 %
#                  exactly is NOT below 5 % (kept); o(6,8) = 12/30; o(7,8) = 0 ->
#                  remove 7.  3 remain.                            kf [3, 6, 8]
SEQ_CELLS = [range(0, 10), range(0, 10), range(5, 15), range(9, 29), range(14, 34),
             range(16, 36), range(10, 40), range(0, 26), range(28, 42)]
SEQ_EVENTS = [(True, []), (False, []), (True, []), (True, []), (True, [0]), (False, []),
              (True, [2]), (True, [4]), (True, [7])]
SEQ_FINAL = [3, 6, 8]


def _seq_pose(f):
    c, s = [(1, 0), (0, 1), (-1, 0), (0, -1)][f % 4]
    T = np.eye(4)
    T[:3, :3] = [[c, -s, 0], [s, c, 0], [0, 0, 1]]
    T[:3, 3] = [f - 3, 2 * f, -1]
    return T


def keyframe_sequence():
    """(clouds [(mu, cov)], poses [F,12]) of the hand-worked sequence."""
    clouds, poses = [], []
    for f, cells in enumerate(SEQ_CELLS):
        T = _seq_pose(f)
        w = np.array([[x + 0.5, 0.5, 0.5] for x in cells])
        local = (w - T[:3, 3]) @ T[:3, :3]          # R^T (w - t), exact
        clouds.append((local.astype(np.float32),
                       np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (len(cells), 1))))
        poses.append(T[:3].reshape(12))
    return clouds, np.stack(poses)


def test_run_keyframes_hand_worked_sequence(oracle):
    clouds, poses = keyframe_sequence()
    maps = [oracle.VoxelMap(mu, cov, 1.0, 1) for mu, cov in clouds]
    kf, events = okf.run_keyframes(clouds, maps, poses, list(range(len(clouds))), 0, n_odom=3)
    assert events == SEQ_EVENTS
    assert kf == SEQ_FINAL


def test_library_host_rules_on_hand_worked_sequence():
    """The library's host-only keyframe entry points (gvox_keyframe_insert_test,
    gvox_keyframe_update_counts: the P:280 insertion test and the removal rules
    formed from raw counts in the C ABI) replay the hand-worked sequence, with
    every count taken from plain set arithmetic on the cells (no GPU)."""
    import paper_2407_10344_b200 as gv
    cells = [set(c) for c in SEQ_CELLS]
    kf, events = [], []
    for f in range(len(cells)):
        if kf:
            cnt = len(cells[f] & set().union(*[cells[k] for k in kf]))
            if not gv.keyframe_insert_test(cnt, len(cells[f])):
                events.append((False, []))
                continue
        ks = kf + [f]
        c = np.array([[len(cells[a] & cells[b]) for b in ks] for a in ks], np.int64)
        rm, o = gv.keyframe_update_counts(c, [len(cells[a]) for a in ks], n_odom=3)
        np.testing.assert_array_equal(o, c / np.array([len(cells[a]) for a in ks])[:, None])
        events.append((True, [ks[a] for a in np.flatnonzero(rm)]))
        kf = [ks[a] for a in range(len(ks)) if not rm[a]]
    assert events == SEQ_EVENTS and kf == SEQ_FINAL


def test_library_insert_test_boundaries_and_errors():
    import paper_2407_10344_b200 as gv
    assert gv.keyframe_insert_test(17, 20) is True       # 85 %
    assert gv.keyframe_insert_test(18, 20) is False      # 90 % is not smaller than 90 %
    assert gv.keyframe_insert_test(0, 0) is False         # empty frame: 0 < 0 is false
    assert gv.keyframe_insert_test(5, 10, 1, 2) is False  # custom threshold 50 %
    for bad in ((-1, 5), (6, 5)):
        with pytest.raises(gv.GvoxError):
            gv.keyframe_insert_test(*bad)
    with pytest.raises(gv.GvoxError):
        gv.keyframe_update_counts([[3, 4], [0, 2]], [3, 2])   # count 4 > size 3
    rm, o = gv.keyframe_update_counts([[0, 0], [0, 0]], [0, 0])
    assert o.tolist() == [[0, 0], [0, 0]] and rm.tolist() == [True, False]
