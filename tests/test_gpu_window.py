"""GPU sliding window (paper_2501_08672_b200.window, csrc/window.cu) against
the reference's own maintain run (tests/golden/window_walk.npz): report
counts, slot layout and rows bit-exact frame by frame, with capacity drops,
init_fn synthesis and device-side optimisation between frames."""
import numpy as np
import pytest
import torch

from window_case import case, init_row, optimise

pytestmark = pytest.mark.gpu


def _setup():
    from paper_2501_08672_b200.voxmap import HashOctree
    from paper_2501_08672_b200.window import GaussianWindow
    d, frames = case()
    K, L, root = int(d["sh_coeffs"]), int(d["max_level"]), float(d["root_len"])
    vmap = HashOctree(root, max_level=L)
    vmap.set_gaussians_dev(d["seeded"], d["seed_rows"])
    win = GaussianWindow(capacity=int(d["capacity"]), sh_coeffs=K)
    return d, frames, K, L, root, vmap, win


class _G:          # Gaussian3D-like payload for init_fn
    def __init__(self, row, K):
        self.mean_w, self.rot, self.scale = row[:3], row[3:12].reshape(3, 3), row[12:15]
        self.opacity, self.sh = float(row[15]), row[16:].reshape(K, 3)


@pytest.mark.parametrize("fov_as", ["tensor", "set", "tensor_dup"])
def test_window_walk_matches_reference(fov_as):
    from paper_2501_08672_b200.voxmap import VoxelKey
    d, frames, K, L, root, vmap, win = _setup()
    for f, fr in enumerate(frames):
        init = (lambda k: [_G(init_row(k, root, L, K), K)]) if f >= 20 else None
        fov = torch.as_tensor(fr["fov"], device="cuda") if fov_as != "set" else \
            {VoxelKey(int(a), int(b), int(c), L) for a, b, c in fr["fov"]}
        if fov_as == "tensor_dup":      # repeated, unordered FoV keys: the same window
            g = torch.Generator().manual_seed(f)
            fov = torch.cat([fov, fov[torch.randperm(fov.shape[0], generator=g).to(fov.device)]])
        rep = win.maintain(vmap, fov, init_fn=init, sensor_pos=fr["sensor"])
        got = [rep.n_live, rep.added, rep.removed, rep.moved, rep.dropped]
        assert got == list(fr["report"]), (f, got, fr["report"])
        win.audit()
        assert np.array_equal(win.live_keys_dev().cpu().numpy(), fr["live"]), f
        rows = win.rows_dev().cpu().numpy()
        assert np.array_equal(rows, fr["rows"]), f
        # the generator's device-side optimisation, applied to the arena
        new = optimise(fr["live"], rows, K)
        n = win.n
        win.shs[:n, 0, 0] = torch.as_tensor(new[:, 16], device="cuda")
        win.opacities[:n] = torch.as_tensor(new[:, 15], device="cuda")


def test_window_renders_from_its_arena():
    """as_gaussian_arrays() is a view of the live prefix the renderer reads."""
    d, frames, K, L, root, vmap, win = _setup()
    fr = frames[0]
    win.maintain(vmap, torch.as_tensor(fr["fov"], device="cuda"), sensor_pos=fr["sensor"])
    ga = win.as_gaussian_arrays()
    assert len(ga) == win.n
    assert ga.means.data_ptr() == win.means.data_ptr()


def test_window_full_without_sensor():
    from paper_2501_08672_b200.errors import WindowFull
    from paper_2501_08672_b200.voxmap import HashOctree
    from paper_2501_08672_b200.window import GaussianWindow
    vmap = HashOctree(1.0, max_level=1)
    keys = np.array([[i, 0, 0] for i in range(8)], dtype=np.int64)
    vmap.set_gaussians_dev(keys, np.ones((8, 19), dtype=np.float32))
    win = GaussianWindow(capacity=4, sh_coeffs=1)
    with pytest.raises(WindowFull):
        win.maintain(vmap, torch.as_tensor(keys, device="cuda"))
