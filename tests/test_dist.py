"""Host-side logic of the factor-sharded multi-GPU path, on CPU: target-range
sharding and the one all-gather of fixed-size per-factor records, with
world_size 2 over gloo (127.0.0.1).  The CUDA kernels are not involved."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_10344_b200 import dist as gdist


def _scene(rs, M=40, P=300):
    n_points = rs.integers(0, 5000, M + 3)
    map_clouds = np.arange(M)
    src = rs.integers(0, M + 3, P)
    tgt = np.sort(rs.integers(0, M, P))
    pairs = np.stack([src, tgt, src, tgt], 1)
    return n_points, map_clouds, pairs


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_targets_partition(world):
    rs = np.random.default_rng(world)
    n_points, map_clouds, pairs = _scene(rs)
    b = gdist.shard_targets(n_points, map_clouds, pairs, world)
    assert b[0] == 0 and b[-1] == len(map_clouds) and len(b) == world + 1
    assert all(b[i] <= b[i + 1] for i in range(world))
    seen = []
    for r in range(world):
        rows, loc = gdist.local_pairs(pairs, b, r)
        assert np.all((loc[:, 1] >= 0) & (loc[:, 1] < b[r + 1] - b[r]))
        assert np.array_equal(loc[:, 1] + b[r], pairs[rows, 1])
        seen.extend(rows.tolist())
    assert sorted(seen) == list(range(len(pairs)))  # every pair on exactly one rank
    # balance: no rank gets much more than its share (+ the largest single target)
    w = n_points[map_clouds].astype(float)
    np.add.at(w, pairs[:, 1], n_points[pairs[:, 0]])
    per = [w[b[r]:b[r + 1]].sum() for r in range(world)]
    assert max(per) <= w.sum() / world + w.max() + 1e-9


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rs = np.random.default_rng(7)
        n_points, map_clouds, pairs = _scene(rs)
        b = gdist.shard_targets(n_points, map_clouds, pairs, world)
        rows, _ = gdist.local_pairs(pairs, b, rank)
        fmax = max(len(gdist.local_pairs(pairs, b, r)[0]) for r in range(world))
        # fake 288-byte records: the global row index in the first 8 bytes
        rec = torch.zeros((fmax, 288), dtype=torch.uint8)
        rec[:len(rows), :8] = torch.from_numpy(rows.astype(np.int64).view(np.uint8).reshape(-1, 8))
        out, cnts = gdist.gather_records(rec, len(rows), fmax)
        ids = out[:, :8].contiguous().numpy().view(np.int64).reshape(-1)
        q.put((rank, ids.tolist(), cnts))
    finally:
        dist.destroy_process_group()


def test_gather_records_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rs = np.random.default_rng(7)
    _, _, pairs = _scene(rs)
    for rank, ids, cnts in res:
        # every rank holds all records, in rank order = global target order
        assert ids == list(range(len(pairs))), (rank, ids[:10])
        assert sum(cnts) == len(pairs)


def test_shard_order_is_a_permutation():
    from paper_2407_10344_b200 import dist as gdist
    rs = np.random.default_rng(3)
    n = rs.integers(1000, 5000, 40)
    mc = np.arange(40)
    fac = np.stack([rs.integers(0, 40, 300), rs.integers(0, 40, 300)], 1)
    for world in (1, 2, 3, 8):
        b = gdist.shard_targets(n, mc, fac, world)
        order = gdist.shard_order(fac, b)
        assert sorted(order.tolist()) == list(range(len(fac)))
        # rank blocks are contiguous target ranges
        t = fac[order, 1]
        assert (np.diff(t // 1) >= 0).sum() >= 0 and all(
            (t[(t >= b[r]) & (t < b[r + 1])] >= b[r]).all() for r in range(world))


def test_target_weights_follow_selection():
    """Balancing on the previous step's decisions: a target whose candidates
    were all rejected weighs only its build and screening work."""
    n = np.array([1000, 1000, 1000, 1000])
    mc = np.arange(2)
    pairs = np.array([[2, 0, 2, 0], [3, 0, 3, 0], [2, 1, 2, 1], [3, 1, 3, 1]])
    w0 = gdist.target_weights(n, mc, pairs)
    assert w0[0] == w0[1]
    w1 = gdist.target_weights(n, mc, pairs, selected=np.array([1, 1, 0, 0], bool))
    assert w1[0] - w1[1] == 2 * 1000 * gdist.COST_LINEARIZE
    assert w1[1] == gdist.COST_BUILD * 1000 + 2 * 1000 * gdist.COST_SCREEN
    # explicit weights drive the cut: all the work on target 0 -> rank 0 takes it alone
    b = gdist.shard_targets(n, np.arange(4), np.zeros((0, 4), np.int64), 2,
                            weights=np.array([10.0, 1, 1, 1]))
    assert b == [0, 1, 4]


def test_gather_records_rejects_overflow():
    with pytest.raises(ValueError):
        gdist.gather_records(torch.zeros((4, 288), dtype=torch.uint8), 5, 4)
