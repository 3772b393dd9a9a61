"""TEST INFRASTRUCTURE ONLY — ctypes loader for the oracle's C restatement.

Builds oracle/build/liboracle_blend.so with oracle/Makefile on first use if it
is missing (gcc is in the image).  Never imported by the product package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "liboracle_blend.so")
_lib = None

_P = ctypes.c_void_p
_I = ctypes.c_int64
_D = ctypes.c_double


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        L.oracle_camera_points.argtypes = [_P, _P, _P, _I, _P]
        L.oracle_csr_count.argtypes = [_P, _I, _I, _I, _P, _P]
        L.oracle_csr_count.restype = _I
        L.oracle_csr_fill.argtypes = [_P, _I, _I, _I, _P, _P, _P, _P]
        L.oracle_forward.argtypes = [_P, _P, _P, _P, _P, _P, _P, _I, _I, _D, _D, _D,
                                     _P, _P, _P, _P, _P, _P]
        L.oracle_backward_entries.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I,
                                              _P, _P, _P]
        L.oracle_accumulate.argtypes = [_P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I,
                                        _D, _P, _P, _P, _P]
        L.oracle_screen_grads.argtypes = [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _D,
                                          _P, _P, _P, _P, _P, _P, _P]
        _lib = L
    return _lib


def ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return ctypes.c_void_p(a.ctypes.data)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)
