"""The CPU restatement of the window protocol (oracle/window.py) against the
reference's own run (tests/golden/window_walk.npz): slot layout, rows and
report counts, frame by frame."""
import numpy as np

from window_case import case, init_row, optimise


def test_oracle_window_matches_reference_walk():
    from oracle.window import Window
    d, frames = case()
    K, L, root = int(d["sh_coeffs"]), int(d["max_level"]), float(d["root_len"])
    store = {tuple(int(v) for v in k): r.copy() for k, r in zip(d["seeded"], d["seed_rows"])}
    win = Window(int(d["capacity"]), 16 + 3 * K)
    for f, fr in enumerate(frames):
        init = (lambda k: init_row(k, root, L, K)) if f >= 20 else None
        rep = win.maintain(store, {tuple(int(v) for v in k) for k in fr["fov"]}, root / (1 << L), init, fr["sensor"])
        assert rep == list(fr["report"]), (f, rep, fr["report"])
        assert win.keys == [tuple(int(v) for v in k) for k in fr["live"]], f
        assert np.array_equal(win.rows[:win.n], fr["rows"]), f
        win.rows[:win.n] = optimise(win.keys, win.rows[:win.n], K)
