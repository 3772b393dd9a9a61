"""The boundary's exception types (errors.py:4-53): same names and bases as
the reference's, and - when the reference package is importable beside this
one - subclasses of the reference's own classes, so existing `except
livsplat.errors.X:` clauses keep catching (CPU only)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"
NAMES = ["BehindCamera", "OutOfBounds", "Degenerate", "MissingVoxel", "WindowFull", "EmptyMask", "MissingCache",
         "NoAssociations", "TooFewPixels", "SingularGain", "NonMonotonicTime"]


def test_same_names_and_builtin_bases():
    from paper_2501_08672_b200 import errors
    want = {"BehindCamera": ValueError, "OutOfBounds": ValueError, "Degenerate": ValueError,
            "MissingVoxel": KeyError, "WindowFull": RuntimeError, "EmptyMask": ValueError,
            "MissingCache": RuntimeError, "NoAssociations": RuntimeError, "TooFewPixels": RuntimeError,
            "SingularGain": RuntimeError, "NonMonotonicTime": ValueError}
    for name, base in want.items():
        assert issubclass(getattr(errors, name), base), name
    assert issubclass(errors.CapacityExceeded, RuntimeError)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")
def test_reference_except_clauses_catch_ours():
    code = ("import livsplat.errors as le\n"
            "from paper_2501_08672_b200 import errors as e\n"
            f"for n in {NAMES!r}:\n"
            "    try:\n"
            "        raise getattr(e, n)('x')\n"
            "    except getattr(le, n):\n"
            "        pass\n"
            "print('ok')\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF_SRC, ROOT]), PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr


def test_host_readable_tensors_convert_for_numpy():
    """RenderOutput's tensors: np.asarray gives a host copy (the reference's
    write_ppm / psnr call np.asarray on render images); torch ops on them
    return plain tensors."""
    import numpy as np
    import torch
    from paper_2501_08672_b200.raster import host_readable
    t = host_readable(torch.arange(12, dtype=torch.float32).reshape(2, 2, 3))
    a = np.asarray(t)
    assert isinstance(a, np.ndarray) and a.dtype == np.float32 and np.array_equal(a, np.arange(12).reshape(2, 2, 3))
    assert np.asarray(t, dtype=float).dtype == np.float64
    assert type(t * 2) is torch.Tensor
    img8 = np.clip(np.round(np.asarray(t) * 255.0), 0, 255).astype(np.uint8)    # raster.py:513
    assert img8.shape == (2, 2, 3)
