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
