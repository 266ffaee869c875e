"""Keyframe mechanism on the CUDA path:
gvox_overlap_union counts bit-exact against the oracle (integers), member
lists longer than one shared-memory chunk (32), empty member lists; the
KeyframeList driver (union test + pair overlaps + gvox_keyframe_update) gives
the same keyframe list and events as the oracle's run over a frame sequence."""
import numpy as np
import pytest

import synth
from oracle import keyframes as okf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx(gv):
    return gv.Context(0)


@pytest.fixture(scope="module")
def scene():
    # 30 frames 0.15 m apart + 20 keyframe clouds 2 m apart (C3 recipe, smaller)
    return synth.smoother_window(n_frames=30, n_kf=20, per_frame=2, n_points=6000, rings=64, az=512)


@pytest.fixture(scope="module")
def built(gv, ctx, oracle, scene):
    sc = scene
    clouds = [gv.Cloud(ctx, *sc.cloud(c)) for c in range(sc.num_clouds)]
    maps = gv.create_voxelmaps(ctx, clouds, sc.r0, sc.levels)
    ocl = [sc.cloud(c) for c in range(sc.num_clouds)]
    omp = [oracle.VoxelMap(*sc.cloud(c)[:2], sc.r0, sc.levels) for c in range(sc.num_clouds)]
    return clouds, maps, ocl, omp


def test_union_overlap_parity(gv, ctx, oracle, scene, built):
    sc = scene
    clouds, maps, ocl, omp = built
    C = sc.num_clouds
    rs = np.random.default_rng(11)
    queries, members = [], []
    for q in range(12):
        k = [0, 1, 3, 20, 33, 49][q % 6]
        mem = rs.choice(C, k, replace=False) if k <= C else rs.integers(0, C, k)
        src = int(rs.integers(0, C))
        queries.append([src, src, len(members), len(mem)])
        members += [[int(m), int(m)] for m in mem]
    for level in range(sc.levels):
        got = gv.overlap_union(ctx, clouds, maps, queries, members, sc.gt_poses, level)
        for q, (src, pi, first, cnt) in enumerate(queries):
            ms = [m for m, _ in members[first:first + cnt]]
            ref = oracle.overlap_union(ocl[src][0], [omp[m] for m in ms], sc.gt_poses[pi],
                                       np.stack([sc.gt_poses[m] for m in ms]) if ms else np.zeros((0, 12)),
                                       level)
            assert int(got[q]) == ref, (level, q, cnt)
    # device output
    import torch
    out = torch.zeros(len(queries), dtype=torch.int32, device="cuda")
    gv.overlap_union(ctx, clouds, maps, queries, members, sc.gt_poses, 1, out=out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(),
                          gv.overlap_union(ctx, clouds, maps, queries, members, sc.gt_poses, 1))


def test_keyframe_list_matches_oracle(gv, ctx, oracle, scene, built):
    sc = scene
    clouds, maps, ocl, omp = built
    # the keyframe clouds in driving order (they were generated backward), then the frames
    seq = list(range(sc.num_clouds - 1, 29, -1)) + list(range(30))
    kl = gv.KeyframeList(ctx, level=sc.overlap_level, n_odom=6)
    events = [kl.add_frame(f, clouds, maps, sc.gt_poses) for f in seq]
    okfs, oev = okf.run_keyframes(ocl, omp, sc.gt_poses, seq, sc.overlap_level, n_odom=6)
    assert [e[0] for e in events] == [e[0] for e in oev]
    assert [sorted(e[1]) for e in events] == [sorted(e[1]) for e in oev]
    assert kl.frames == okfs
    assert sum(e[0] for e in events) > 6 and any(e[1] for e in events)  # both rules exercised


def test_keyframe_list_hand_worked_sequence(gv, ctx):
    """KeyframeList (GPU union and pair overlaps + the C-ABI rules) replays the
    hand-worked sequence of tests/test_oracle_keyframes.py."""
    from tests.test_oracle_keyframes import SEQ_EVENTS, SEQ_FINAL, keyframe_sequence
    clouds_h, poses = keyframe_sequence()
    clouds = [gv.Cloud(ctx, mu, cov) for mu, cov in clouds_h]
    maps = gv.create_voxelmaps(ctx, clouds, 1.0, 1)
    kl = gv.KeyframeList(ctx, level=0, n_odom=3)
    events = [kl.add_frame(f, clouds, maps, poses) for f in range(len(clouds))]
    assert [(bool(a), list(b)) for a, b in events] == SEQ_EVENTS
    assert kl.frames == SEQ_FINAL
