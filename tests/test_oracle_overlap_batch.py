"""Pins of the oracle's batched overlap (oracle_overlap_batch, P:280 overlap
rate, P:391 global-factor screening), CPU only.

The batch routine feeds bench.py's cpu_baseline and the --impl reference arm,
so each of its indices is pinned against something other than itself:

* every count equals a brute-force membership count: the pair's relative pose
  T_j^-1 T_i composed in plain numpy (tests/se3.py), every source point
  transformed in numpy and looked up in the target map one by one (the lookup
  is pinned by a brute-force containing-cell scan in test_oracle_voxelmap.py);
* the batch is built so that a swapped pair column (source <-> target), a
  swapped pose column (pose_i <-> pose_j) or a pose taken from the wrong pair
  changes the count: clouds of different sizes and distinct poses;
* hand-counted values on an exact lattice (one point per cell, integer
  translations): the overlap of a translated copy is the number of shared
  cells, in both directions of a size-asymmetric pair;
* thread count does not change the result.
"""
import numpy as np
import pytest

from tests.se3 import rel_pose, to12


def _lattice_cloud(cells):
    """One point at the centre of each unit cell (r = 1)."""
    mu = np.array([[x + 0.5, y + 0.5, z + 0.5] for x, y, z in cells], np.float32)
    cov = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (len(cells), 1))
    return mu, cov


def _brute_count(oracle, mu, vmap, Ti, Tj, level):
    T = np.asarray(rel_pose(Ti, Tj)).reshape(3, 4)
    q = mu.astype(np.float64) @ T[:, :3].T + T[:, 3]
    return int(sum(vmap.lookup(level, p) >= 0 for p in q))


def test_overlap_batch_hand_counted_lattice(oracle):
    # A: cells x = 0..9 (10 points); B: cells x = 0..3 (4 points).  Poses are
    # pure integer translations, so the overlap is the count of shared cells.
    A = _lattice_cloud([(x, 0, 0) for x in range(10)])
    B = _lattice_cloud([(x, 0, 0) for x in range(4)])
    maps = [oracle.VoxelMap(*A, 1.0, 1), oracle.VoxelMap(*B, 1.0, 1)]

    def tr(x):
        T = np.eye(4)
        T[0, 3] = x
        return to12(T)

    poses = np.stack([tr(0), tr(2), tr(7)])
    pairs = np.array([
        [0, 1, 0, 0],   # A -> B, same pose: A's cells 0..3 lie in B: 4
        [1, 0, 0, 0],   # B -> A, same pose: all 4 of B's cells lie in A: 4
        [0, 1, 1, 0],   # A at +2 -> B at 0: world 2..11 vs 0..3 -> {2, 3}: 2
        [0, 1, 0, 1],   # A at 0 -> B at +2: world 0..9 vs 2..5 -> 4
        [1, 0, 2, 0],   # B at +7 -> A at 0: world 7..10 vs 0..9 -> {7, 8, 9}: 3
        [1, 0, 0, 2],   # B at 0 -> A at +7: world 0..3 vs 7..16 -> 0
        [0, 0, 1, 2],   # A at +2 -> A at +7: world 2..11 vs 7..16 -> 7..11: 5
        [0, 0, 2, 1],   # A at +7 -> A at +2: 7..16 vs 2..11 -> 5
    ], np.int64)
    want = [4, 4, 2, 4, 3, 0, 5, 5]
    got = oracle.overlap_batch([A[0], B[0]], maps, pairs, poses, 0)
    assert got.tolist() == want
    # the pose is a parameter, not an index into the pair list
    got_threads = oracle.overlap_batch([A[0], B[0]], maps, pairs, poses, 0, num_threads=3)
    assert got_threads.tolist() == want


@pytest.mark.parametrize("level", [0, 1])
def test_overlap_batch_brute_force_random(oracle, level):
    rs = np.random.default_rng(280)
    sizes = [300, 180, 240]
    clouds = []
    for n in sizes:
        mu = rs.uniform(-4, 4, (n, 3)).astype(np.float32)
        cov = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (n, 1))
        clouds.append((mu, cov))
    maps = [oracle.VoxelMap(mu, cov, 0.5, 2) for mu, cov in clouds]
    # four distinct poses close enough to overlap partially
    poses = []
    for k in range(4):
        T = np.eye(4)
        a = 0.3 * k
        T[:3, :3] = [[np.cos(a), -np.sin(a), 0], [np.sin(a), np.cos(a), 0], [0, 0, 1]]
        T[:3, 3] = rs.normal(0, 0.8, 3)
        poses.append(to12(T))
    poses = np.stack(poses)
    pairs = []
    for s in range(3):
        for t in range(3):
            for pi in range(4):
                pj = (pi + 1 + s + t) % 4
                pairs.append([s, t, pi, pj])
    pairs = np.array(pairs, np.int64)
    got = oracle.overlap_batch([c[0] for c in clouds], maps, pairs, poses, level, num_threads=4)
    want = [_brute_count(oracle, clouds[s][0], maps[t], poses[pi], poses[pj], level)
            for s, t, pi, pj in pairs]
    assert got.tolist() == want
    # the fixture discriminates the columns: swapping any pair of columns
    # changes at least one count
    for perm in ([1, 0, 2, 3], [0, 1, 3, 2]):
        sw = pairs[:, perm]
        alt = [_brute_count(oracle, clouds[s][0], maps[t], poses[pi], poses[pj], level)
               for s, t, pi, pj in sw]
        assert alt != want
    assert min(want) >= 0 and max(want) > 0


def test_overlap_batch_empty_source_and_empty_batch(oracle):
    mu, cov = _lattice_cloud([(0, 0, 0), (1, 0, 0)])
    m = oracle.VoxelMap(mu, cov, 1.0, 1)
    empty = np.zeros((0, 3), np.float32)
    I = np.eye(4)[:3].reshape(1, 12)
    got = oracle.overlap_batch([empty, mu], [m], np.array([[0, 0, 0, 0], [1, 0, 0, 0]]), I, 0)
    assert got.tolist() == [0, 2]
    assert oracle.overlap_batch([mu], [m], np.zeros((0, 4), np.int64), I, 0).tolist() == []
