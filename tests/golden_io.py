"""Loading helpers for the committed golden fixtures (tests/golden/*.npz).

The fixtures were produced by the reference itself (tools/make_golden.py);
this module only unpacks them into the oracle's / the package's input form.
"""
import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def case_inputs(d):
    P = {k: d[k] for k in ("means", "rots", "scales", "opacities", "shs")}
    R_wc, t_wc = d["R_wc"], d["t_wc"]
    R_cw = R_wc.T
    t_cw = -R_cw @ t_wc          # SE3.inverse (geometry.py:151-153)
    fx, fy, cx, cy, w, h = d["cam"]
    cam = SimpleNamespace(fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))
    st = SimpleNamespace(**{k[3:]: (d[k].item() if d[k].ndim == 0 else d[k])
                           for k in d if k.startswith("st_")})
    st.sh_degree = int(st.sh_degree)
    return P, R_cw, t_cw, cam, st


RENDER_CASES = [f"rand{s}_cut{c}" for s in range(4) for c in (0, 1)] + [
    "odd_cut0", "odd_cut1", "room_v0_cut1", "room_v1_cut0", "room_v2_cut1"]
