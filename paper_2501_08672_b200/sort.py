"""Device sort and grouping primitives of the map / window paths (csrc/sort.cu).

sort_pairs: stable LSD radix sort of int64 keys (optionally with int32
values; by default the permutation), the stable lexsort voxmap.py:213-230
and the window's key grouping use.  segments: run starts of a sorted key
array (np.diff / unique on the reference side).  No library sort is used.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Tuple

import torch

from . import _lib

_SIGN = -(1 << 63)


def _temp(n: int, device) -> torch.Tensor:
    nb = ctypes.c_size_t()
    _lib.check(_lib.load().lsb_sort_temp_bytes(int(n), ctypes.byref(nb)), "sort_temp_bytes")
    return torch.empty(max(nb.value, 1), dtype=torch.uint8, device=device)


def sort_pairs(keys: torch.Tensor, vals: Optional[torch.Tensor] = None, key_bits: int = 64,
               signed: bool = True, stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """(sorted keys int64, values int32 in the same order).  Stable: equal
    keys keep their input order.  `signed`: int64 order (the sign bit is
    flipped for the unsigned digit passes); key_bits counts the low bits
    that vary (64 when signed)."""
    _lib.require()
    keys = keys.reshape(-1).to(torch.int64).contiguous()
    n = keys.numel()
    dev = keys.device
    if signed:
        kin = keys ^ _SIGN
        key_bits = 64
    else:
        kin = keys
    kout = torch.empty_like(kin)
    vout = torch.empty(n, dtype=torch.int32, device=dev)
    vin = None if vals is None else vals.reshape(-1).to(torch.int32).contiguous()
    if n:
        tmp = _temp(n, dev)
        _lib.check(_lib.load().lsb_sort_pairs(
            ctypes.c_void_p(kin.data_ptr()), ctypes.c_void_p(vin.data_ptr()) if vin is not None else None,
            ctypes.c_void_p(kout.data_ptr()), ctypes.c_void_p(vout.data_ptr()), n, int(key_bits),
            ctypes.c_void_p(tmp.data_ptr()), tmp.numel(), _lib.stream_ptr(stream)), "sort_pairs")
    return (kout ^ _SIGN if signed else kout), vout


def segments(sorted_keys: torch.Tensor, stream=None) -> torch.Tensor:
    """Start index (int64) of every run of equal keys in a sorted array
    (one host sync for the count)."""
    _lib.require()
    k = sorted_keys.reshape(-1).to(torch.int64).contiguous()
    n = k.numel()
    starts = torch.empty(max(n, 1), dtype=torch.int64, device=k.device)
    nseg = torch.zeros(1, dtype=torch.int64, device=k.device)
    tmp = _temp(n, k.device)
    _lib.check(_lib.load().lsb_segments(ctypes.c_void_p(k.data_ptr()), n, ctypes.c_void_p(starts.data_ptr()),
                                        ctypes.c_void_p(nseg.data_ptr()), ctypes.c_void_p(tmp.data_ptr()),
                                        tmp.numel(), _lib.stream_ptr(stream)), "segments")
    return starts[: int(nseg.item())]


def unique_sorted(sorted_keys: torch.Tensor, stream=None) -> torch.Tensor:
    """The distinct keys of a sorted array, ascending."""
    return sorted_keys.reshape(-1)[segments(sorted_keys, stream)]
