"""The library's own device sort and grouping (csrc/sort.cu) against numpy:
stable radix sort of int64 keys (the stable lexsort of voxmap.py:213-230),
run starts of sorted keys (np.unique)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,span,seed", [(1, 5, 0), (33, 4, 1), (4095, 1000, 2), (4097, 3, 3), (100_000, 1 << 40, 4),
                                         (250_001, 70, 5)])
def test_sort_pairs_is_numpys_stable_argsort(n, span, seed):
    import torch
    from paper_2501_08672_b200.sort import sort_pairs
    rng = np.random.default_rng(seed)
    keys = rng.integers(-span, span, n, dtype=np.int64)
    k, perm = sort_pairs(torch.as_tensor(keys, device="cuda"))
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(perm.cpu().numpy(), order)
    assert np.array_equal(k.cpu().numpy(), keys[order])


def test_sort_pairs_values_and_unsigned_bits():
    import torch
    from paper_2501_08672_b200.sort import sort_pairs
    rng = np.random.default_rng(7)
    keys = rng.integers(0, 1 << 20, 50_000, dtype=np.int64)
    vals = rng.integers(-1000, 1000, 50_000).astype(np.int32)
    k, v = sort_pairs(torch.as_tensor(keys, device="cuda"), torch.as_tensor(vals, device="cuda"), key_bits=20,
                      signed=False)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(k.cpu().numpy(), keys[order])
    assert np.array_equal(v.cpu().numpy(), vals[order])


@pytest.mark.parametrize("n", [1, 7, 4096, 4097, 123_457])
def test_segments_are_numpy_unique(n):
    import torch
    from paper_2501_08672_b200.sort import segments, unique_sorted
    rng = np.random.default_rng(n)
    keys = np.sort(rng.integers(-50, 50, n, dtype=np.int64) * 7919)
    st = segments(torch.as_tensor(keys, device="cuda")).cpu().numpy()
    u, first = np.unique(keys, return_index=True)
    assert np.array_equal(st, first)
    assert np.array_equal(unique_sorted(torch.as_tensor(keys, device="cuda")).cpu().numpy(), u)


def test_empty_inputs():
    import torch
    from paper_2501_08672_b200.sort import segments, sort_pairs
    k, v = sort_pairs(torch.empty(0, dtype=torch.int64, device="cuda"))
    assert k.numel() == 0 and v.numel() == 0
    assert segments(torch.empty(0, dtype=torch.int64, device="cuda")).numel() == 0
