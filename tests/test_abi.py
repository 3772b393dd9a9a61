"""CPU checks of the C-ABI boundary: the library loads and exports every
symbol include/lsb.h declares (no compute calls; no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "lsb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lsb_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("lsb_render_fwd", "lsb_render_bwd", "lsb_workspace_bytes", "lsb_photometric_loss"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2501_08672_b200 import _lib

    if not os.path.exists(_lib.SO_PATH):
        pytest.skip("libsplat_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.SO_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(declared_functions()) <= bound, set(declared_functions()) - bound


def test_workspace_query_without_gpu():
    from paper_2501_08672_b200 import _lib

    if not os.path.exists(_lib.SO_PATH):
        pytest.skip("libsplat_b200.so not built")
    lib = _lib.load()
    assert lib.lsb_abi_version() == 1
    d = _lib.Dims(1000, 64, 48, 1, 16, 1 << 16)
    nb = ctypes.c_size_t()
    assert lib.lsb_workspace_bytes(ctypes.byref(d), ctypes.byref(nb)) == 0
    assert nb.value > 1000 * 64
    bad = _lib.Dims(1000, 64, 48, 1, 8, 1 << 16)
    assert lib.lsb_workspace_bytes(ctypes.byref(bad), ctypes.byref(nb)) == _lib.LSB_EINVAL
    assert b"tile" in lib.lsb_last_error()
