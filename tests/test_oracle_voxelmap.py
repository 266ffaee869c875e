"""Pins of the oracle's voxelmap, lookup and overlap (CPU only).

Each pin checks the oracle against something other than itself: hand-computed
cases, brute-force binning, a brute-force containing-cell
scan (reading Q8), floor semantics on exact boundaries,
level monotonicity and insertion-order independence, and the
overlap identities self = 1, disjoint = 0, half = 0.5.
"""
import numpy as np
import pytest

from tests.se3 import random_pose, to12, to44

HALF = 1 << 20


def unpack(key):
    key = int(key)
    return ((key >> 42) & 0x1FFFFF) - HALF, ((key >> 21) & 0x1FFFFF) - HALF, (key & 0x1FFFFF) - HALF


def brute_bin(mu, cov, r):
    """Brute-force binning: dict (kx,ky,kz) -> [sum mu, sum cov, n]."""
    out = {}
    for p, c in zip(mu.astype(np.float64), cov.astype(np.float64)):
        k = tuple(int(np.floor(x / r)) for x in p)
        a = out.setdefault(k, [np.zeros(3), np.zeros(6), 0])
        a[0] += p
        a[1] += c
        a[2] += 1
    return out


def rand_cloud(rs, n, scale=10.0):
    mu = rs.uniform(-scale, scale, (n, 3)).astype(np.float32)
    A = rs.normal(0, 1, (n, 3, 3))
    C = A @ A.transpose(0, 2, 1) + 0.1 * np.eye(3)
    cov = np.stack([C[:, 0, 0], C[:, 0, 1], C[:, 0, 2], C[:, 1, 1], C[:, 1, 2], C[:, 2, 2]], 1)
    return mu, cov.astype(np.float32)


def test_single_point_one_voxel_per_level(oracle):
    mu = np.array([[1.3, -2.7, 0.4]], np.float32)
    cov = np.array([[1, 0.1, 0.2, 2, 0.3, 3]], np.float32)
    m = oracle.VoxelMap(mu, cov, 0.5, 3)
    for l in range(3):
        keys, means, covs, counts = m.export(l)
        assert len(keys) == 1 and counts[0] == 1
        np.testing.assert_array_equal(means[0], mu[0].astype(np.float64))
        np.testing.assert_array_equal(covs[0], cov[0].astype(np.float64))
        r = 0.5 * 2 ** l
        assert unpack(keys[0]) == tuple(int(np.floor(float(x) / r)) for x in mu[0])


def test_two_points_midpoint_and_average_covariance(oracle):
    mu = np.array([[0.25, 0.25, 0.25], [0.75, 0.5, 0.125]], np.float32)
    cov = np.array([[1, 0, 0, 1, 0, 1], [3, 1, 0, 5, 0, 7]], np.float32)
    m = oracle.VoxelMap(mu, cov, 1.0, 1)
    keys, means, covs, counts = m.export(0)
    assert counts.tolist() == [2]
    np.testing.assert_array_equal(means[0], [0.5, 0.375, 0.1875])
    np.testing.assert_array_equal(covs[0], [2, 0.5, 0, 3, 0, 4])


@pytest.mark.parametrize("seed", [0, 1])
def test_brute_force_binning_1k(oracle, seed):
    rs = np.random.default_rng(seed)
    mu, cov = rand_cloud(rs, 1000, 3.0)
    r0, L = 0.5, 3
    m = oracle.VoxelMap(mu, cov, r0, L)
    for l in range(L):
        bf = brute_bin(mu, cov, r0 * 2 ** l)
        keys, means, covs, counts = m.export(l)
        assert len(keys) == len(bf)
        assert np.all(np.diff(keys) > 0), "canonical order = ascending packed key"
        for key, mean, c, n in zip(keys, means, covs, counts):
            s_mu, s_cov, bn = bf[unpack(key)]
            assert n == bn
            np.testing.assert_allclose(mean, s_mu / bn, rtol=0, atol=1e-12)
            np.testing.assert_allclose(c, s_cov / bn, rtol=1e-12, atol=1e-12)


def test_boundary_floor_semantics(oracle):
    # coordinates exactly on multiples of r go to the higher-index voxel
    mu = np.array([[1.0, 2.0, -1.0], [0.999999, 1.999999, -1.000001]], np.float32)
    cov = np.tile(np.array([1, 0, 0, 1, 0, 1], np.float32), (2, 1))
    m = oracle.VoxelMap(mu, cov, 1.0, 1)
    keys, _, _, _ = m.export(0)
    got = sorted(unpack(k) for k in keys)
    assert got == sorted([(1, 2, -1), (0, 1, -2)])
    # lookups at exact boundaries
    assert m.lookup(0, [1.0, 2.0, -1.0]) == oracle.pack_key(1, 2, -1)
    assert m.lookup(0, [1.0, 2.0, -0.5]) == oracle.pack_key(1, 2, -1)
    assert m.lookup(0, [1.0, 2.0, 0.0]) == -1  # z = 0 is the next cell up


def test_level_monotonicity_and_order_independence(oracle):
    rs = np.random.default_rng(5)
    mu, cov = rand_cloud(rs, 3000, 8.0)
    m = oracle.VoxelMap(mu, cov, 0.25, 4)
    counts = [m.num_voxels(l) for l in range(4)]
    assert all(counts[l] <= counts[l - 1] for l in range(1, 4))
    perm = rs.permutation(len(mu))
    m2 = oracle.VoxelMap(mu[perm], cov[perm], 0.25, 4)
    for l in range(4):
        a, b = m.export(l), m2.export(l)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[3], b[3])
        np.testing.assert_allclose(a[1], b[1], rtol=0, atol=1e-12)
        np.testing.assert_allclose(a[2], b[2], rtol=1e-12, atol=1e-12)


def test_empty_cloud_and_range_errors(oracle):
    m = oracle.VoxelMap(np.zeros((0, 3), np.float32), np.zeros((0, 6), np.float32), 1.0, 2)
    assert m.num_voxels(0) == 0 and m.num_voxels(1) == 0
    with pytest.raises(ValueError, match="out of range"):
        oracle.VoxelMap(np.array([[3e6, 0, 0]], np.float32), np.ones((1, 6), np.float32), 1.0, 1)
    with pytest.raises(ValueError):
        oracle.VoxelMap(np.zeros((1, 3), np.float32), np.ones((1, 6), np.float32), 0.0, 1)
    with pytest.raises(ValueError):
        oracle.VoxelMap(np.zeros((1, 3), np.float32), np.ones((1, 6), np.float32), 1.0, 9)


def test_lookup_brute_force_containing_cell(oracle):
    rs = np.random.default_rng(7)
    mu, cov = rand_cloud(rs, 200, 2.0)
    r0, L = 0.5, 2
    m = oracle.VoxelMap(mu, cov, r0, L)
    qs = rs.uniform(-2.5, 2.5, (500, 3))
    for l in range(L):
        r = r0 * 2 ** l
        keys = m.export(l)[0]
        cells = [unpack(k) for k in keys]
        for q in qs:
            hit = [k for k, c in zip(keys, cells)
                   if all(c[a] * r <= q[a] < (c[a] + 1) * r for a in range(3))]
            assert len(hit) <= 1
            assert m.lookup(l, q) == (int(hit[0]) if hit else -1)


def test_overlap_self_disjoint_half(oracle):
    rs = np.random.default_rng(11)
    mu, cov = rand_cloud(rs, 2000, 5.0)
    m = oracle.VoxelMap(mu, cov, 1.0, 2)
    I = to12(np.eye(4))
    for l in range(2):
        assert oracle.overlap(mu, m, I, I, l) == len(mu)  # self overlap = 1.0
    # the same cloud with an arbitrary common world pose: still 1.0
    T = random_pose(rs, 0.3, 3.0)
    assert oracle.overlap(mu, m, T, T, 0) == len(mu)
    # disjoint: source shifted far away
    Tf = to44(I)
    Tf[0, 3] = 100.0
    assert oracle.overlap(mu, m, to12(Tf), I, 0) == 0
    # half translated: a cloud filling every 1 m cell of x in [-5,5),
    # y, z in [-2,2) (4 points per cell); shifting by +5 m along x moves the
    # x >= 0 half outside the map's extent
    g = np.stack(np.meshgrid(np.arange(-5, 5), np.arange(-2, 2), np.arange(-2, 2),
                             indexing="ij"), -1).reshape(-1, 3)
    dense = (np.repeat(g, 4, 0) + rs.uniform(0.05, 0.95, (len(g) * 4, 3))).astype(np.float32)
    md = oracle.VoxelMap(dense, np.tile(cov[:1], (len(dense), 1)), 1.0, 1)
    Th = to44(I)
    Th[0, 3] = 5.0
    cnt = oracle.overlap(dense, md, to12(Th), I, 0)
    # brute-force membership: transformed key in the set of occupied keys
    keys = set(int(k) for k in md.export(0)[0])
    q = dense.astype(np.float64) + np.array([5.0, 0, 0])
    bf = sum(1 for p in q if oracle.pack_key(*[int(np.floor(x)) for x in p]) in keys)
    assert cnt == bf
    assert abs(cnt / len(dense) - 0.5) <= 1.0 / len(dense)


def test_overlap_empty_source(oracle):
    mu = np.zeros((0, 3), np.float32)
    rs = np.random.default_rng(1)
    tm, tc = rand_cloud(rs, 10)
    m = oracle.VoxelMap(tm, tc, 1.0, 1)
    I = to12(np.eye(4))
    assert oracle.overlap(mu, m, I, I, 0) == 0
