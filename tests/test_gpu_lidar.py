"""Plane fits and the LiDAR point-to-plane measurement on the GPU
(csrc/voxmap.cu) against the reference's own outputs (tests/golden/lidar.npz)
and the CPU restatement.  Bars: validity flags exact; normals / centroids to
1e-9 (f64 Jacobi vs LAPACK on the same statistics); z to 1e-9; H and the
pose block of H^T R^-1 H / H^T R^-1 z within 1e-3 relative (BASELINE.json)."""
import numpy as np
import pytest
import torch

from golden_io import load

pytestmark = pytest.mark.gpu


def _map(d):
    from paper_2501_08672_b200.voxmap import HashOctree
    m = HashOctree(float(d["root_len"]), max_level=int(d["max_level"]))
    m.accumulate_points_dev(torch.as_tensor(d["points"], device="cuda"))
    return m


def test_fit_planes_match_reference():
    d = load("lidar")
    m = _map(d)
    nrm, anc, ok = (t.cpu().numpy() for t in m.fit_planes_dev(d["keys"], d["origin"]))
    assert np.array_equal(ok, d["valid"])
    assert np.abs(nrm[ok] - d["normals"][ok]).max() <= 1e-9
    assert np.abs(anc[ok] - d["anchors"][ok]).max() <= 1e-9
    assert np.isnan(nrm[~ok]).all()


def test_lidar_measurement_matches_reference():
    from paper_2501_08672_b200.estimator import FilterConfig, NavState, lidar_measurement
    from paper_2501_08672_b200.geometry import SE3
    d = load("lidar")
    m = _map(d)
    meas = lidar_measurement(NavState(SE3(d["T_wi_R"], d["T_wi_t"])), d["points_l"], m,
                             SE3(d["T_il_R"], d["T_il_t"]), FilterConfig(lidar_gate=float(d["lidar_gate"])))
    assert len(meas.z) == len(d["z"])
    assert np.abs(meas.z - d["z"]).max() <= 1e-9
    H6 = meas.H[:, :6]
    assert np.abs(H6 - d["H6"]).max() / np.abs(d["H6"]).max() <= 1e-3
    assert not np.any(meas.H[:, 6:])
    # device H/b against H^T R^-1 H, H^T R^-1 z of the reference's rows
    A, b = meas.hb()
    inv = 1.0 / float(d["lidar_sigma"]) ** 2
    A_ref = d["H6"].T @ d["H6"] * inv
    b_ref = d["H6"].T @ d["z"] * inv
    assert np.abs(A - A_ref).max() / np.abs(A_ref).max() <= 1e-3
    assert np.abs(b - b_ref).max() / np.abs(b_ref).max() <= 1e-3


def test_lidar_no_associations():
    from paper_2501_08672_b200.errors import NoAssociations
    from paper_2501_08672_b200.estimator import FilterConfig, NavState, lidar_measurement
    from paper_2501_08672_b200.geometry import SE3
    from paper_2501_08672_b200.voxmap import HashOctree
    m = HashOctree(0.4, max_level=2)
    m.accumulate_points_dev(torch.zeros((1, 3), dtype=torch.float64, device="cuda"))
    with pytest.raises(NoAssociations):
        lidar_measurement(NavState(), np.array([[5.0, 5.0, 5.0]]), m, SE3.identity(), FilterConfig())
