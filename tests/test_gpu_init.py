"""Batched Gaussian initialisation (paper_2501_08672_b200.initialize,
csrc/voxmap.cu k_init_gaussians) against the reference's own per-leaf loop
(tests/golden/init.npz, tools/make_golden_init.py): which leaves get a
Gaussian exactly; rows to f32 round-off (means exact, normal / colour from
f64 Jacobi vs LAPACK and f64 bilinear sums within 1e-6)."""
import numpy as np
import pytest
import torch

from golden_io import load

pytestmark = pytest.mark.gpu


def test_insert_new_gaussians_matches_reference():
    from types import SimpleNamespace
    from paper_2501_08672_b200.geometry import SE3
    from paper_2501_08672_b200.initialize import insert_new_gaussians
    from paper_2501_08672_b200.voxmap import HashOctree
    d = load("init")
    m = HashOctree(0.4, max_level=2)
    m.accumulate_points_dev(torch.as_tensor(d["scan0"], device="cuda"))
    m.set_gaussians_dev(d["keys0"], np.ones((len(d["keys0"]), 19), dtype=np.float32))
    fx, fy, cx, cy, w, h = d["cam"]
    cam = SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))
    keys, rows, made = insert_new_gaussians(m, d["scan1"], d["image"], SE3(d["R_wc"], d["t_wc"]), cam, d["origin"],
                                            kappa=float(d["kappa"]), delta=float(d["delta"]),
                                            opacity=float(d["opacity"]), near=float(d["near"]))
    assert np.array_equal(keys.cpu().numpy(), d["gkeys"])
    made = made.cpu().numpy()
    assert np.array_equal(made, d["created"])
    got = rows.cpu().numpy()[made]
    ref = d["rows"][made].astype(np.float32)
    assert np.array_equal(got[:, 0:3], ref[:, 0:3])            # means: the scan centroid, f32
    assert np.abs(got - ref).max() <= 1e-6
    # the new Gaussians are in the map's store
    stored = m.gaussian_rows_dev(d["gkeys"][made]).cpu().numpy()
    assert np.array_equal(stored, got)
