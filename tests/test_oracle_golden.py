"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden/).

CPU-only.  Discrete results (visible ids, bboxes, depth order, per-pixel
counts, CSR lists) must match bit for bit; floating outputs to round-off,
since the reference kernels run numba fastmath and the oracle plain C.
"""
import numpy as np
import pytest

from golden_io import RENDER_CASES, case_inputs, load
from oracle import raster as orc


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-30)


@pytest.fixture(scope="module", params=RENDER_CASES)
def case(request):
    d = load(request.param)
    P, R_cw, t_cw, cam, st = case_inputs(d)
    c = orc.render(P, R_cw, t_cw, cam, st)
    return d, c


def test_camera_points_match_numpy_blas(case):
    d, c = case
    P, R_cw, t_cw, _, _ = case_inputs(d)
    ref = P["means"] @ R_cw.T + t_cw   # raster.py:137 as the reference evaluates it
    assert np.array_equal(orc.camera_points(P["means"], R_cw, t_cw), ref)


def test_preprocess_discrete_bit_exact(case):
    d, c = case
    assert np.array_equal(c["ids"], d["ids"])
    assert np.array_equal(c["bboxes"], d["bboxes"])
    assert np.array_equal(c["mu_c"], d["mu_c"])          # sort keys: bit-exact


def test_preprocess_float(case):
    d, c = case
    assert rel(c["mu_i"], d["mu_i"]) <= 1e-13
    assert rel(c["conics"], d["conics"]) <= 1e-12
    assert rel(c["colors"], d["colors"]) <= 1e-13
    assert np.array_equal(c["interior"], d["interior"])


def test_csr_bit_exact(case):
    d, c = case
    assert np.array_equal(c["offsets"], d["offsets"])
    assert np.array_equal(c["entry_splat"], d["entry_splat"])


def test_forward_matches_reference(case):
    d, c = case
    assert np.abs(c["image"] - d["image"]).max() <= 1e-9
    assert np.abs(c["t_final"].reshape(d["t_final"].shape) - d["t_final"]).max() <= 1e-9
    assert np.array_equal(c["n_proc"].reshape(d["n_proc"].shape), d["n_proc"])


def test_backward_matches_reference(case):
    d, c = case
    out = orc.backward(c, d["grad_image"], d["R_ic"], d["t_ic"])
    g = out["grads"]
    for k, gk in (("mean", "g_mean"), ("rot", "g_rot"), ("scale", "g_scale"),
                  ("opacity", "g_opacity"), ("sh", "g_sh")):
        assert rel(g[k], d[gk]) <= 1e-8, k
    p = out["pose"]
    for k, gk in (("rho", "p_rho"), ("tau", "p_tau"), ("camera_rho", "p_crho"),
                  ("camera_tau", "p_ctau")):
        assert rel(p[k], d[gk]) <= 1e-8, k


def test_pose_rows_match_reference(case):
    d, c = case
    rows = orc.pose_rows(c, d["pix_ids"], d["R_ic"], d["t_ic"])
    assert rel(rows, d["pose_rows"]) <= 1e-8


def test_tile_lists_reproduce_reference_csr(case):
    """Per pixel, the tile list filtered by bbox membership equals the
    reference's CSR list — entry for entry."""
    d, c = case
    ranges, entries, gid = orc.tile_lists(c)
    cam = c["cam"]
    tx_n = (cam.width + 15) // 16
    bb = c["bboxes"]
    rng = np.random.default_rng(0)
    npx = cam.width * cam.height
    for p in rng.choice(npx, size=min(400, npx), replace=False):
        y, x = divmod(int(p), cam.width)
        t = (y // 16) * tx_n + x // 16
        lst = entries[ranges[t, 0]:ranges[t, 1]]
        inside = lst[(bb[lst, 0] <= x) & (x < bb[lst, 1]) & (bb[lst, 2] <= y) & (y < bb[lst, 3])]
        ref = d["entry_splat"][d["offsets"][p]:d["offsets"][p + 1]]
        assert np.array_equal(inside, ref)


def test_adam_update_matches_reference():
    from oracle.optim import Adam
    d = load("adam")
    a = Adam({"x": (50, 3)})
    for g, ref in zip(d["grads"], d["steps"]):
        a.step += 1
        assert np.array_equal(a.update("x", g, 1e-3), ref)


def test_optimize_window_matches_reference():
    from types import SimpleNamespace
    from oracle.optim import optimize_views
    d = load("optimize_plane")
    n = len(d["in_means"])
    P = {"means": d["in_means"].astype(float), "rots": d["in_rots"].astype(float).reshape(n, 3, 3),
         "scales": d["in_scales"].astype(float), "opacities": d["in_opacities"].astype(float),
         "shs": d["in_shs"].astype(float)}
    fx, fy, cx, cy, w, h = d["cam"]
    cam = SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))
    st = SimpleNamespace(near=0.01, dilation=0.3, alpha_clamp=0.99, transmittance_min=1e-4, footprint_sigma=6.0,
                         alpha_cut=0.0, max_footprint_px=512.0, background=np.zeros(3), sh_degree=0)
    out, hist = optimize_views(P, [d["observed"]], [(np.eye(3), np.zeros(3))], cam, st, 10)
    assert np.abs(np.array(hist)[:, 0] - d["loss"]).max() <= 1e-9
    for k in ("means", "scales", "opacities", "shs"):
        assert np.abs(out[k].astype(np.float32) - d["out_" + k]).max() <= 1e-6, k
    assert np.abs(out["rots"].reshape(n, 9).astype(np.float32) - d["out_rots"]).max() <= 1e-6


def test_voxmap_oracle_matches_reference():
    from oracle.voxmap import Map, keys
    d = load("voxmap")
    rl, L = float(d["root_len"]), int(d["max_level"])
    assert np.array_equal(keys(d["pts"], rl), d["root_keys"][:, :3])
    assert np.array_equal(keys(d["pts"], rl / (1 << L)), d["leaf_keys"][:, :3])
    m = Map(rl, L)
    m.accumulate_points(d["pts"])
    sk = [tuple(k[:3]) for k in d["stat_keys"]]
    assert set(sk) == set(m.leaves)
    for i, k in enumerate(sk):
        leaf = m.leaves[k]
        assert leaf[0] == d["stat_count"][i]
        assert np.allclose(leaf[1], d["stat_sum"][i], rtol=1e-12, atol=1e-12)
        assert np.allclose(leaf[2], d["stat_outer"][i], rtol=1e-12, atol=1e-12)
    rng = np.random.default_rng(11)
    rng.uniform(-3, 3, size=(4000, 3)); rng.normal(scale=0.05, size=(1000, 3))
    for p in rng.uniform(-2, 2, size=(600, 3)):
        m.try_insert(p)
    it = m.iter_keys()
    assert np.array_equal(np.array(it), d["iter_keys"][:, :3])
    assert np.array_equal(np.array([m.leaves[k][3] for k in it]), d["iter_has_g"])
    assert m.leaf_keys_under_roots(d["fov_roots"]) == {tuple(k[:3]) for k in d["fov_keys"]}
