"""Golden fixture for the map snapshot (LSMAP001) and PLY writers
(voxmap.py:360-415), produced by the REFERENCE in this container.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_snapshot.py

The map holds the window golden's seeded Gaussians (tests/golden/
window_walk.npz: 339 leaves of a 0.8 m / max_level 1 map, K = 4) plus, to
exercise negative keys and several roots, the same rows shifted to negative
coordinates.  Recorded: the snapshot bytes and the PLY text.
"""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from livsplat.geometry import Gaussian3D  # noqa: E402
from livsplat.voxmap import HashOctree, VoxelKey  # noqa: E402

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(HERE, "tests", "golden", "snapshot.npz")


def main():
    w = np.load(os.path.join(HERE, "tests", "golden", "window_walk.npz"))
    keys = np.concatenate([w["seeded"], -w["seeded"] - 1])
    rows = np.concatenate([w["seed_rows"], w["seed_rows"][::-1]])
    m = HashOctree(root_len=0.8, max_level=1, leaf_capacity=1)
    for k, r in zip(keys, rows.astype(np.float64)):
        g = Gaussian3D(mean_w=r[0:3], rot=r[3:12].reshape(3, 3), scale=r[12:15], opacity=float(r[15]),
                       sh=r[16:].reshape(-1, 3), level=1)
        m.ensure_leaf(VoxelKey(int(k[0]), int(k[1]), int(k[2]), 1)).gaussians = [g]
    with tempfile.TemporaryDirectory() as d:
        m.save(os.path.join(d, "map.bin"))
        m.export_ply(os.path.join(d, "map.ply"))
        snap = open(os.path.join(d, "map.bin"), "rb").read()
        ply = open(os.path.join(d, "map.ply"), "rb").read()
    np.savez_compressed(OUT, keys=keys, rows=rows, snapshot=np.frombuffer(snap, dtype=np.uint8),
                        ply=np.frombuffer(ply, dtype=np.uint8))
    print("wrote", OUT, len(snap), "snapshot bytes,", len(ply), "ply bytes")


if __name__ == "__main__":
    main()
