"""bin_mode 1 (contributing tile lists, include/lsb.h) on the CPU oracle.

The mode drops a (tile, splat) pair only when the splat's alpha >= alpha_cut
ellipse misses every pixel of the tile.  Checked here against the reference's
own per-entry alphas (the oracle forward's scratch, _kernels.py:104-108): every
CSR entry the reference composites (alpha >= cut) must keep its tile, and the
kept lists must be a depth-ordered subsequence of the full bbox lists.
"""
import numpy as np
import pytest

from golden_io import case_inputs, load

CUT_CASES = [f"rand{s}_cut1" for s in range(4)] + ["odd_cut1", "room_v0_cut1", "room_v2_cut1"]


@pytest.mark.parametrize("name", CUT_CASES)
def test_contributing_lists_are_conservative(name):
    from oracle import raster as orc
    d = load(name)
    P, R_cw, t_cw, cam, st = case_inputs(d)
    c = orc.render(P, R_cw, t_cw, cam, st)
    rows = orc.contributing_tile_rows(c)
    ntx = (cam.width + 15) // 16
    keep = set()
    for s, rs in enumerate(rows):
        for ty, a, b in rs:
            keep.update((ty * ntx + tx, s) for tx in range(a, b + 1))
    # entries the reference composited (alpha >= cut; the scratch holds 0 for skipped ones)
    hit = c["a_scr"] >= st.alpha_cut                    # pixel-major entries (CSR order)
    pix = np.repeat(np.arange(cam.width * cam.height), np.diff(c["offsets"]))[hit]
    tiles = (pix // cam.width // 16) * ntx + (pix % cam.width) // 16
    spl = c["entry_splat"][hit]
    missing = [(int(t), int(s)) for t, s in zip(tiles, spl) if (int(t), int(s)) not in keep]
    assert not missing, f"{len(missing)} composited entries lost their tile, e.g. {missing[:3]}"
    # subsequence of the full lists, same per-tile order
    full_r, full_e, _ = orc.tile_lists(c)
    cr, ce, _ = orc.contributing_tile_lists(c)
    assert len(ce) <= len(full_e)
    for t in range(len(full_r)):
        f = list(full_e[full_r[t, 0]:full_r[t, 1]])
        k = list(ce[cr[t, 0]:cr[t, 1]])
        it = iter(f)
        assert all(x in it for x in k), t


def test_contributing_lists_drop_entries_on_the_room():
    from oracle import raster as orc
    d = load("room_v2_cut1")
    P, R_cw, t_cw, cam, st = case_inputs(d)
    c = orc.render(P, R_cw, t_cw, cam, st)
    _, full_e, _ = orc.tile_lists(c)
    _, ce, _ = orc.contributing_tile_lists(c)
    assert len(ce) < len(full_e)
