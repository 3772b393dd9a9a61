"""Map snapshot (LSMAP001) and PLY export from the device store, against the
reference's own files (tests/golden/snapshot.npz, tools/make_golden_snapshot.py):
byte-identical snapshot, text-identical PLY, lossless load round trip."""
import numpy as np
import pytest

from golden_io import load

pytestmark = pytest.mark.gpu


def _map():
    from paper_2501_08672_b200.voxmap import HashOctree
    d = load("snapshot")
    m = HashOctree(0.8, max_level=1)
    m.set_gaussians_dev(d["keys"], d["rows"])
    return d, m


def test_snapshot_bytes_match_reference(tmp_path):
    d, m = _map()
    p = tmp_path / "map.bin"
    m.save(p)
    assert p.read_bytes() == d["snapshot"].tobytes()
    assert m.gaussian_count() == len(d["keys"])


def test_ply_matches_reference(tmp_path):
    d, m = _map()
    p = tmp_path / "map.ply"
    m.export_ply(p)
    assert p.read_bytes() == d["ply"].tobytes()


def test_snapshot_round_trip(tmp_path):
    from paper_2501_08672_b200.voxmap import HashOctree
    d = load("snapshot")
    p = tmp_path / "ref.bin"
    p.write_bytes(d["snapshot"].tobytes())
    m = HashOctree.load(p)
    q = tmp_path / "again.bin"
    m.save(q)
    assert q.read_bytes() == d["snapshot"].tobytes()
    rows = m.gaussian_rows_dev(d["keys"]).cpu().numpy()
    assert np.array_equal(rows, d["rows"])
    # the loaded map's FoV (its Gaussian-leaf key list) covers every stored leaf
    from paper_2501_08672_b200.voxmap import VoxelKey
    keys = np.asarray(d["keys"], np.int64).reshape(-1, 3)
    roots = {tuple(int(v) for v in (k >> m.max_level)) for k in keys}
    got = m.leaf_keys_under_roots([VoxelKey(a, b, c, 0) for a, b, c in roots])
    assert {k[:3] for k in got} == {tuple(int(v) for v in k) for k in keys}


def test_snapshot_rejects_other_files(tmp_path):
    from paper_2501_08672_b200.voxmap import HashOctree
    p = tmp_path / "x.bin"
    p.write_bytes(b"NOTAMAP!" + bytes(40))
    with pytest.raises(ValueError):
        HashOctree.load(p)
