"""The oracle against the worked values of tests/golden/worked_examples.json
(each with its citation).  The CUDA path is checked against the same fixtures
in tests/test_gpu_parity.py."""
import json
import os

import numpy as np
import pytest

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


@pytest.mark.parametrize("name", ["d2d_unit", "d2d_rotated"])
def test_oracle_d2d_golden(oracle, name):
    g = GOLDEN[name]
    m = oracle.VoxelMap(np.array(g["target_mu"], np.float32), np.array(g["target_cov"], np.float32),
                        g["r0"], g["levels"])
    r = oracle.linearize(np.array(g["source_mu"], np.float32), np.array(g["source_cov"], np.float32),
                         None, m, g["T_i"], g["T_j"])
    assert r["e"] == pytest.approx(g["e"], rel=1e-15)


def test_oracle_voxel_golden(oracle):
    g = GOLDEN["two_points_voxel"]
    m = oracle.VoxelMap(np.array(g["mu"], np.float32), np.array(g["cov"], np.float32), g["r0"], 1)
    keys, means, covs, counts = m.export(0)
    assert keys.tolist() == [oracle.pack_key(*g["voxel_key_xyz"])]
    assert means[0].tolist() == g["mean"] and covs[0].tolist() == g["cov_mean"]
    assert counts.tolist() == [g["count"]]


def test_oracle_visibility_golden(oracle):
    g = GOLDEN["visibility_wall"]
    mu = np.array([g["point"]], np.float32)
    unit = np.array([[1, 0, 0, 1, 0, 1]], np.float32)
    for x, inv in zip(g["viewer_x"], g["invisible"]):
        Tj = np.array([1, 0, 0, x, 0, 1, 0, 0, 0, 0, 1, 0], float)
        m = oracle.VoxelMap(mu - np.array([[x, 0, 0]], np.float32), unit, 1.0, 1)
        r = oracle.linearize(mu, unit, np.array([g["normal"]], np.float32), m,
                             np.eye(4)[:3].reshape(-1), Tj, validate=True)
        assert r["num_invisible"] == inv
