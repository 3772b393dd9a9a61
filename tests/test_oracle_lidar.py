"""Plane fits and the LiDAR measurement restated on the CPU
(oracle/lidar.py) against the reference's own outputs (tests/golden/lidar.npz)."""
import numpy as np

from golden_io import load


def _stats(d):
    from oracle import lidar as orl
    leaf = float(d["root_len"]) / (1 << int(d["max_level"]))
    return orl.leaf_stats(d["points"], leaf), leaf


def test_oracle_fit_planes_match_reference():
    from oracle import lidar as orl
    d = load("lidar")
    stats, _ = _stats(d)
    keys = [tuple(int(v) for v in k) for k in d["keys"]]
    fits = orl.fit_planes(stats, keys, d["origin"])
    valid = np.array([fits[k] is not None for k in keys])
    assert np.array_equal(valid, d["valid"])
    nrm = np.array([fits[k][0] for k, ok in zip(keys, valid) if ok])
    anc = np.array([fits[k][1] for k, ok in zip(keys, valid) if ok])
    assert np.abs(nrm - d["normals"][valid]).max() <= 1e-9
    assert np.abs(anc - d["anchors"][valid]).max() <= 1e-12


def test_oracle_lidar_measurement_matches_reference():
    from oracle import lidar as orl
    d = load("lidar")
    stats, leaf = _stats(d)
    z, H, kept = orl.lidar_measurement(stats, leaf, d["points_l"], d["T_il_R"], d["T_il_t"], d["T_wi_R"],
                                       d["T_wi_t"], float(d["lidar_gate"]))
    assert len(z) == len(d["z"])
    assert np.abs(z - d["z"]).max() <= 1e-9
    assert np.abs(H - d["H6"]).max() <= 1e-9
