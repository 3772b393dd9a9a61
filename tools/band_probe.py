"""Probe: alpha_cut band statistics (tiles re-blended, pairs decided in f64)
per view of a workload, and the kernel time of one view's render."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2501_08672_b200.raster import GaussianArrays, RasterSettings, render
from tools.scene import bake_room, camera_for, orbit_views

for name, v_s, W, H in (("cfg2", 0.0723, 1280, 1024), ("target", 0.0457, 1280, 1024)):
    m, r, s, o, sh = bake_room(v_s)
    a = GaussianArrays(m, r, s, o, sh)
    cam = camera_for(W, H)
    for bm in (0, 1):
        tot = np.zeros(3, int)
        err = 0.0
        for T in orbit_views(10):
            out = render(a, T, cam, RasterSettings(alpha_cut=1 / 255), bin_mode=bm)
            st = out.cache.band_stats()
            tot += np.array(st[:3])
            err = max(err, st[3])
        print(name, "bin_mode", bm, "per 10 views: entries flagged, band pairs, composited =", tot.tolist(),
              "max rel f32 alpha error in band = %.3g" % err, flush=True)
