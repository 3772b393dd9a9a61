"""GPU voxel map vs the reference (voxmap.py): keys bit-exact, leaf sets and
the iteration order exact, leaf statistics to f64 round-off."""
import numpy as np
import pytest

from golden_io import load

pytestmark = pytest.mark.gpu


def _map():
    from paper_2501_08672_b200.voxmap import HashOctree
    d = load("voxmap")
    return d, HashOctree(float(d["root_len"]), int(d["max_level"]), capacity=1 << 12)


def test_keys_bit_exact():
    from paper_2501_08672_b200.voxmap import keys_of_points_dev
    d = load("voxmap")
    rl, L = float(d["root_len"]), int(d["max_level"])
    assert np.array_equal(keys_of_points_dev(d["pts"], rl).cpu().numpy(), d["root_keys"][:, :3])
    assert np.array_equal(keys_of_points_dev(d["pts"], rl / (1 << L)).cpu().numpy(), d["leaf_keys"][:, :3])


def test_reference_key_known_answers():
    from paper_2501_08672_b200.voxmap import VoxelKey, hash_key, leaf_key
    assert hash_key([0.5, 0.5, 0.5], 1.0) == VoxelKey(0, 0, 0, 0)
    assert hash_key([-0.1, 2.3, 0.0], 1.0) == VoxelKey(-1, 2, 0, 0)
    assert hash_key([0.13, 0.0, -0.05], 0.06) == VoxelKey(2, 0, -1, 0)
    assert leaf_key([0.9, 0.1, 0.1], 1.0, 2) == VoxelKey(3, 0, 0, 2)


def test_accumulate_points_matches_reference():
    d, m = _map()
    touched = m.accumulate_points(d["pts"])      # also exercises the rehash growth path
    ref_keys = {tuple(k[:3]) for k in d["stat_keys"]}
    assert {k[:3] for k in touched} == ref_keys
    # every leaf: counts exact, sums / outer products to f64 round-off (the
    # reference's numpy pairwise / BLAS order vs scan order)
    cnt, sm, outer = (t.cpu().numpy() for t in m.leaf_stats_dev(d["stat_keys"][:, :3]))
    assert np.array_equal(cnt, d["stat_count"])
    assert np.allclose(sm, d["stat_sum"], rtol=1e-12, atol=1e-12)
    assert np.allclose(outer, d["stat_outer"], rtol=1e-12, atol=1e-12)
    from paper_2501_08672_b200.voxmap import VoxelKey
    k = d["stat_keys"][5]
    st = m.leaf_stats(VoxelKey(int(k[0]), int(k[1]), int(k[2]), int(d["max_level"])))
    assert st[0] == cnt[5] and np.array_equal(st[1], sm[5]) and np.array_equal(st[2], outer[5])


def test_accumulate_is_deterministic():
    """The leaf statistics are bit-identical across runs (exact fixed-point
    group sums with integer atomics; no floating-point atomics)."""
    import torch
    d = load("voxmap")
    out = []
    for _ in range(2):
        from paper_2501_08672_b200.voxmap import HashOctree
        m = HashOctree(float(d["root_len"]), max_level=int(d["max_level"]))
        for chunk in np.array_split(d["pts"], 3):
            m.accumulate_points_dev(chunk)
        out.append(tuple(t.cpu().numpy() for t in m.leaf_stats_dev(d["stat_keys"][:, :3])))
        torch.cuda.synchronize()
    for a, b in zip(*out):
        assert np.array_equal(a, b)


def test_try_insert_iter_order_and_fov_match_reference():
    from paper_2501_08672_b200.voxmap import VoxelKey
    d, m = _map()
    m.accumulate_points(d["pts"])
    rng = np.random.default_rng(11)
    rng.uniform(-3, 3, size=(4000, 3)); rng.normal(scale=0.05, size=(1000, 3))   # replay the generator
    means = rng.uniform(-2, 2, size=(600, 3))
    m.try_insert_batch(means)
    keys = m.iter_leaf_keys()
    assert np.array_equal(np.array([k[:3] for k in keys]), d["iter_keys"][:, :3])
    has_g = np.array([m.get_leaf(k)["gid"] >= 0 for k in keys])
    assert np.array_equal(has_g, d["iter_has_g"])
    roots = [VoxelKey(int(a), int(b), int(c), 0) for a, b, c, _ in d["fov_roots"]]
    fov = m.leaf_keys_under_roots(roots)
    assert {k[:3] for k in fov} == {tuple(k[:3]) for k in d["fov_keys"]}


def test_try_insert_capacity_one():
    from paper_2501_08672_b200.voxmap import Full, HashOctree, Inserted

    class G:
        def __init__(self, p):
            self.mean_w = np.asarray(p, float)
            self.level = 0
    m = HashOctree(root_len=1.0, max_level=1)
    assert isinstance(m.try_insert(G([0.1, 0.1, 0.1])), Inserted)
    assert isinstance(m.try_insert(G([0.2, 0.2, 0.2])), Full)
    assert isinstance(m.try_insert(G([0.9, 0.1, 0.1])), Inserted)


def test_fov_list_survives_growth_and_store_writes():
    """The FoV walks the map's list of Gaussian leaves (gkeys): Gaussians made
    by try_insert, by set_gaussians_dev (new leaves and replacements, with a
    repeated key) and a table growth (rehash) in between must leave it equal
    to the brute-force set of Gaussian leaves under the roots
    (leaf_keys_under_roots, voxmap.py:232-251)."""
    import torch
    from paper_2501_08672_b200.voxmap import HashOctree, VoxelKey
    rng = np.random.default_rng(5)
    m = HashOctree(0.5, max_level=2, capacity=1 << 10)
    m.try_insert_batch(rng.uniform(-2, 2, size=(300, 3)))
    m.accumulate_points(rng.uniform(-4, 4, size=(20000, 3)))        # grows the table (rehash)
    assert m.cap > 1 << 10
    L = m.max_level
    new_keys = np.floor(rng.uniform(-4, 4, size=(200, 3)) / m.leaf_len).astype(np.int64)
    new_keys = np.concatenate([new_keys, new_keys[:7]])             # repeated keys in one call
    m.set_gaussians_dev(new_keys, np.zeros((len(new_keys), 19), np.float32))
    m.try_insert_batch(rng.uniform(-3, 3, size=(300, 3)))
    keys, slots = m.dump_dev()
    g = m.gslot[slots].cpu().numpy()
    gk = keys.cpu().numpy()[g >= 0]
    assert int(m.n_gkeys.item()) == len(gk)
    roots = {tuple(int(v) for v in r) for r in np.floor(rng.uniform(-4, 4, size=(60, 3)) / m.root_len).astype(np.int64)}
    want = {tuple(int(v) for v in k) for k in gk if (int(k[0]) >> L, int(k[1]) >> L, int(k[2]) >> L) in roots}
    got = m.leaf_keys_under_roots([VoxelKey(a, b, c, 0) for a, b, c in roots])
    assert {k[:3] for k in got} == want and len(want) > 0
    torch.cuda.synchronize()
