"""Factor-sharded linearization on one GPU with 2 ranks (gloo plumbing): the
gathered compact records equal the single-process batch bit for bit, because a
factor's tiling and reduction order depend on the factor alone."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2407_10344_b200 as gv
        from paper_2407_10344_b200 import dist as gdist
        import synth
        sc = synth.make("C4", n_submaps=24, half_blocks=3, n_points=20000)
        ctx = gv.Context(0)
        clouds = gv.create_clouds(ctx, sc.mu, sc.cov, sc.nrm, sc.offsets)
        n = np.diff(sc.offsets)
        fac = sc.factors
        b = gdist.shard_targets(n, sc.map_clouds, fac, world)
        rows, loc = gdist.local_pairs(fac, b, rank)
        maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds[b[rank]:b[rank + 1]]],
                                   sc.r0, sc.levels)
        fmax = max(len(gdist.local_pairs(fac, b, r)[0]) for r in range(world))
        acc = gv.device_records(ctx, fmax, gv.FACTOR_ACCUM_DTYPE)
        gv.linearize_batch_accum(ctx, clouds, maps, loc, sc.poses, out=acc[:len(loc)])
        torch.cuda.synchronize()
        out, cnts = gdist.gather_records(acc, len(loc), fmax)
        # NEXT-4 on N ranks: sharded linearization + one gather + replicated solve
        fixed = np.zeros(len(sc.poses), np.uint8)
        fixed[0] = 1
        delta, res, order = gdist.global_step_sharded(ctx, clouds, maps, fac, b, rank, sc.poses, fixed,
                                                      fmax, tol=1e-10, max_iterations=1000)
        torch.cuda.synchronize()
        q.put((rank, out.cpu().numpy().tobytes(), cnts, delta.cpu().numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def test_sharded_equals_single(gv):
    import torch.multiprocessing as mp
    import synth
    ctx = gv.Context(0)
    sc = synth.make("C4", n_submaps=24, half_blocks=3, n_points=20000)
    clouds = gv.create_clouds(ctx, sc.mu, sc.cov, sc.nrm, sc.offsets)
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    ref = gv.linearize_batch_accum(ctx, clouds, maps, sc.factors, sc.poses)
    assert len(sc.factors) > 20
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_2407_10344_b200 import dist as gdist
    b = gdist.shard_targets(np.diff(sc.offsets), sc.map_clouds, sc.factors, 2)
    order = np.concatenate([gdist.local_pairs(sc.factors, b, r)[0] for r in range(2)])
    want = ref[order].tobytes()  # gathered rows are in shard (target-range) order
    # the single-process step on the same records in the same order
    import torch
    fixed = np.zeros(len(sc.poses), np.uint8)
    fixed[0] = 1
    ref_acc = torch.from_numpy(np.ascontiguousarray(ref[order]).view(np.uint8).reshape(len(order), -1)).cuda()
    d_ref, _, _, _ = gv.solve_global(ctx, sc.factors[order], ref_acc, sc.poses, fixed, tol=1e-10,
                                     max_iterations=1000)
    torch.cuda.synchronize()
    for rank, blob, cnts, dblob in res:
        assert sum(cnts) == len(sc.factors)
        assert blob == want, f"rank {rank}: gathered records differ from the single batch"
        assert dblob == d_ref.cpu().numpy().tobytes(), f"rank {rank}: sharded global step differs"


def _nccl_worker(port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        import paper_2407_10344_b200 as gv
        from paper_2407_10344_b200 import dist as gdist
        import synth
        assert dist.get_backend() == "nccl"
        sc = synth.make("C4", n_submaps=24, half_blocks=3, n_points=20000)
        ctx = gv.Context(0)
        clouds = gv.create_clouds(ctx, sc.mu, sc.cov, sc.nrm, sc.offsets)
        fac = sc.factors
        b = gdist.shard_targets(np.diff(sc.offsets), sc.map_clouds, fac, 1)
        maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
        fmax = gdist.max_count(len(fac), ctx.device)
        acc = gv.device_records(ctx, fmax, gv.FACTOR_ACCUM_DTYPE)
        gv.linearize_batch_accum(ctx, clouds, maps, fac, sc.poses, out=acc[:len(fac)])
        out, cnts = gdist.gather_records(acc, len(fac), fmax)       # the NCCL collective
        fixed = np.zeros(len(sc.poses), np.uint8)
        fixed[0] = 1
        delta, res, order = gdist.global_step_sharded(ctx, clouds, maps, fac, b, 0, sc.poses, fixed,
                                                      None, tol=1e-10, max_iterations=1000)
        torch.cuda.synchronize()
        q.put((out.cpu().numpy().tobytes(), cnts, delta.cpu().numpy().tobytes(), order.tolist()))
    finally:
        dist.destroy_process_group()


def test_nccl_world1_gather_and_global_step(gv):
    """The NCCL backend actually executes the gather (world size 1 on the one
    GPU of the box): the records come back bitwise, with the count header, and
    the sharded global step equals the single-process step."""
    import torch
    import torch.multiprocessing as mp
    import synth
    ctx = gv.Context(0)
    sc = synth.make("C4", n_submaps=24, half_blocks=3, n_points=20000)
    clouds = gv.create_clouds(ctx, sc.mu, sc.cov, sc.nrm, sc.offsets)
    maps = gv.create_voxelmaps(ctx, [clouds[int(c)] for c in sc.map_clouds], sc.r0, sc.levels)
    ref = gv.linearize_batch_accum(ctx, clouds, maps, sc.factors, sc.poses)
    fixed = np.zeros(len(sc.poses), np.uint8)
    fixed[0] = 1
    ref_acc = torch.from_numpy(np.ascontiguousarray(ref).view(np.uint8).reshape(len(ref), -1)).cuda()
    d_ref, _, _, _ = gv.solve_global(ctx, sc.factors, ref_acc, sc.poses, fixed, tol=1e-10,
                                     max_iterations=1000)
    torch.cuda.synchronize()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    p = mpc.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    blob, cnts, dblob, order = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert cnts == [len(sc.factors)] and order == list(range(len(sc.factors)))
    assert blob == ref.tobytes()
    assert dblob == d_ref.cpu().numpy().tobytes()
