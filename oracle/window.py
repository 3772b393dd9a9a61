"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's sliding-window
maintain protocol (livsplat window.py:136-276), pinned against
tests/golden/window_walk.npz (produced by the reference itself,
tools/make_golden_window.py).  Keys are (ix, iy, iz) tuples at the map's leaf
level; the map's Gaussians are a dict key -> f32 arena row
(mean 3 | rot 9 | scale 3 | opacity 1 | sh 3K, window.py:58-60).
"""
from __future__ import annotations

import numpy as np


class Window:
    def __init__(self, capacity: int, row_floats: int):
        self.capacity = capacity
        self.rows = np.zeros((capacity, row_floats), dtype=np.float32)
        self.keys: list = []            # slot -> key (live prefix)

    @property
    def n(self) -> int:
        return len(self.keys)

    def maintain(self, store: dict, fov: set, edge: float, init_fn=None, sensor=None):
        """Returns [n_live, added, removed, moved, dropped] (window.py:254-276)."""
        live = {k: s for s, k in enumerate(self.keys)}
        delete = sorted(set(live) - fov)                       # window.py:136-143
        add = sorted(fov - set(live))
        for k in delete:                                        # window.py:145-150
            store[k] = self.rows[live[k]].copy()
        marks = sorted(live[k] for k in delete)                 # window.py:151-181
        dele = set(marks)
        rear, moved = self.n - 1, 0
        for d in marks:
            while rear in dele and rear > d:
                rear -= 1
            if rear <= d:
                break
            self.rows[d] = self.rows[rear]
            self.keys[d] = self.keys[rear]
            rear -= 1
            moved += 1
        n = self.n - len(marks)
        self.keys = self.keys[:n]
        dropped = 0
        if n + len(add) > self.capacity:                         # window.py:262-270
            if sensor is None:
                raise RuntimeError("capacity exceeded and no sensor position to rank drops")
            room = self.capacity - n
            origin = np.asarray(sensor, dtype=float)
            ranked = sorted(add, key=lambda k: (float(np.linalg.norm((np.array(k, dtype=float) + 0.5) * edge
                                                                     - origin)), k))
            dropped = len(add) - room
            add = sorted(ranked[:room])
        rows = []                                               # window.py:183-209
        for k in add:
            if k in store:
                rows.append((k, store[k]))
            elif init_fn is not None:
                r = init_fn(k)
                if r is not None:
                    store[k] = r
                    rows.append((k, r))
        if n + len(rows) > self.capacity:
            raise RuntimeError("WindowFull")
        for k, r in rows:
            self.rows[len(self.keys)] = r
            self.keys.append(k)
        return [self.n, len(rows), len(delete), moved, dropped]
