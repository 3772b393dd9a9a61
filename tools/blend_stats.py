"""Work statistics of the blend on one view (CPU, oracle restatement): how
many of the (pixel, tile entry) pairs the tile-warps evaluate can composite
(alpha >= cut inside the bbox), at pixel / lane-run / half-tile / tile-row
granularity, and how many the reference actually processes before the
pixel's transmittance terminates.  Guides the blend's skip tests.

    python tools/blend_stats.py [v_s] [view] [W H]
"""
import sys
from types import SimpleNamespace

import numpy as np

sys.path.insert(0, ".")
from oracle import raster as orc  # noqa: E402
from tools.scene import bake_room, camera_for, orbit_views  # noqa: E402


def main():
    v_s = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0457
    view = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    W, H = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (1280, 1024)
    m, r, s, o, sh = bake_room(v_s)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    P = {"means": f32(m), "rots": f32(r), "scales": f32(s), "opacities": f32(o), "shs": f32(sh)}
    cam = camera_for(W, H)
    T_cw = orbit_views(10)[view].inverse()
    st = SimpleNamespace(near=0.01, dilation=0.3, alpha_clamp=0.99, transmittance_min=1e-4, footprint_sigma=6.0,
                         alpha_cut=1 / 255, max_footprint_px=512.0, background=np.zeros(3), sh_degree=0)
    cache = orc.render(P, T_cw.R, T_cw.t, cam, st)
    rows = orc.contributing_tile_rows(cache)
    ntx = (W + 15) // 16
    ent_s, ent_t = [], []
    for sidx, rs in enumerate(rows):
        for ty, a, b in rs:
            for tx in range(a, b + 1):
                ent_s.append(sidx)
                ent_t.append(ty * ntx + tx)
    ent_s, ent_t = np.array(ent_s), np.array(ent_t)
    I = len(ent_s)
    mu, con, op, bb = cache["mu_i"], cache["conics"], cache["opac"], cache["bboxes"]
    yy, xx = np.mgrid[0:16, 0:16]
    stats = dict(pairs=0, inbox=0, take=0, run_any=0, half_any=0, half_inbox=0, quarter_any=0, row_any=0)
    for c0 in range(0, I, 20000):
        s_, t_ = ent_s[c0:c0 + 20000], ent_t[c0:c0 + 20000]
        px = (t_ % ntx)[:, None, None] * 16 + xx[None]
        py = (t_ // ntx)[:, None, None] * 16 + yy[None]
        dx = px - mu[s_, 0][:, None, None]
        dy = py - mu[s_, 1][:, None, None]
        q = con[s_, 0][:, None, None] * dx * dx + 2 * con[s_, 1][:, None, None] * dx * dy + \
            con[s_, 2][:, None, None] * dy * dy
        al = np.minimum(op[s_][:, None, None] * np.exp(-0.5 * q), st.alpha_clamp)
        inb = (px >= bb[s_, 0][:, None, None]) & (px < bb[s_, 1][:, None, None]) & \
              (py >= bb[s_, 2][:, None, None]) & (py < bb[s_, 3][:, None, None]) & (px < W) & (py < H)
        tk = inb & (al >= st.alpha_cut)
        stats["pairs"] += tk.size
        stats["inbox"] += int(inb.sum())
        stats["take"] += int(tk.sum())
        # lane runs: 4 px wide, rows r and r+8 -> per (row, 4-col group)
        stats["run_any"] += int(tk.reshape(-1, 16, 4, 4).any(axis=3).sum())
        stats["half_any"] += int(tk.reshape(-1, 2, 8, 16).any(axis=(2, 3)).sum())
        stats["half_inbox"] += int(inb.reshape(-1, 2, 8, 16).any(axis=(2, 3)).sum())
        stats["quarter_any"] += int(tk.reshape(-1, 4, 4, 16).any(axis=(2, 3)).sum())
        stats["row_any"] += int(tk.any(axis=2).sum())
    n_proc = int(cache["n_proc"].sum())
    print(f"view {view}: M={len(bb)} I={I} pairs={stats['pairs']:,}")
    print(f"  in bbox            {stats['inbox'] / stats['pairs']:.3f}")
    print(f"  alpha >= cut       {stats['take'] / stats['pairs']:.3f}")
    print(f"  processed (ref, T) {n_proc / stats['pairs']:.3f}  (entries in bbox before termination)")
    print(f"  4-px runs with a take      {stats['run_any'] / (I * 64):.3f}")
    print(f"  pixel rows with a take     {stats['row_any'] / (I * 16):.3f}")
    print(f"  4-row quarters with a take {stats['quarter_any'] / (I * 4):.3f}")
    print(f"  8-row halves with a take   {stats['half_any'] / (I * 2):.3f}   halves in bbox {stats['half_inbox'] / (I * 2):.3f}")


if __name__ == "__main__":
    main()


def composited(cache):
    """Pairs the reference composites (alpha >= cut, before termination)."""
    off, npr, a = cache["offsets"], cache["n_proc"], cache["a_scr"]
    idx = np.arange(len(a))
    pix = np.repeat(np.arange(len(npr)), np.diff(off))
    processed = idx - off[pix] < npr[pix]
    return int((processed & (a >= cache["st"].alpha_cut)).sum()), int(processed.sum())
