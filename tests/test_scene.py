"""The restated scene generator reproduces the reference's bake_scene."""
import numpy as np

from golden_io import load


def test_bake_room_matches_reference_fixture():
    from tools.scene import bake_room
    d = load("scene_room_0323")
    m, r, s, o, sh = bake_room(0.323)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)
    assert len(m) == len(d["means"]) == 9896
    assert np.array_equal(f32(m), d["means"])
    assert np.array_equal(f32(r), d["rots"])
    assert np.array_equal(f32(s), d["scales"])
    assert np.array_equal(f32(o), d["opacities"])
    assert np.abs(f32(sh) - d["shs"]).max() <= 1e-6


def test_room_sizes_match_survey():
    from tools.scene import bake_room
    assert len(bake_room(0.0723)[0]) == 203877
