"""Inputs of the window golden case (tests/golden/window_walk.npz; generator:
tools/make_golden_window.py, which runs the reference)."""
import numpy as np

from golden_io import load


def case():
    d = load("window_walk")
    F = len(d["n"])
    frames = []
    for f in range(F):
        fov = d["fov"][d["fov_off"][f]:d["fov_off"][f + 1]]
        live = d["live"][d["live_off"][f]:d["live_off"][f + 1]]
        rows = d["rows"][d["live_off"][f]:d["live_off"][f + 1]]
        frames.append(dict(fov=fov, sensor=d["sensor"][f], live=live, rows=rows, report=d["report"][f]))
    return d, frames


def init_row(key, root_len, max_level, K):
    """The generator's init_gaussian (deterministic per key) as an f32 row."""
    edge = root_len / (1 << max_level)
    c = (np.array(key[:3], dtype=float) + 0.5) * edge
    s = 0.001 * (key[0] + 10 * key[1] + 100 * key[2] + 1)
    f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
    return np.concatenate([f32(c), np.eye(3).ravel(), f32([1e-3, 0.1 + s, 0.1]), [0.5],
                           f32(np.full((K, 3), s)).ravel()]).astype(np.float32)


def optimise(keys, rows, K):
    """The generator's device-side step between frames (f32 arithmetic)."""
    rows = rows.copy()
    ix = np.asarray(keys)[:, 0]
    rows[:, 16] = rows[:, 16] + (0.01 * (ix + 1)).astype(np.float32)          # shs[slot, 0, 0]
    rows[:, 15] = rows[:, 15] * np.float32(0.99)                                # opacity
    return rows
