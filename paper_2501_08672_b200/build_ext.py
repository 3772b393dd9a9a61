"""Build libsplat_b200.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsplat_b200.so")
BUILD = os.path.join(HERE, "csrc", "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
          "-Xptxas", "-v", "--expt-relaxed-constexpr"]
# per-file extra flags: the preprocess keeps f64 rounding where numpy rounds
EXTRA = {"preprocess.cu": ["--fmad=false"], "adam.cu": ["--fmad=false"]}
SOURCES = ["preprocess.cu", "blend.cu", "chain.cu", "loss.cu", "adam.cu", "pose.cu", "voxmap.cu", "window.cu",
           "ieskf.cu", "sort.cu", "api.cu"]


def build(verbose: bool = False, defines=(), out: str = OUT, tag: str = "") -> str:
    """Compile every source for sm_100a and link `out`.  `defines` (e.g.
    ["FWD_MIN_BLOCKS=7"]) and `tag` build tuning variants side by side."""
    bdir = BUILD + (("_" + tag) if tag else "")
    os.makedirs(bdir, exist_ok=True)
    objs = []
    dflags = [f"-D{d}" for d in defines]
    for src in SOURCES:
        obj = os.path.join(bdir, src.replace(".cu", ".o"))
        srcp = os.path.join(CSRC, src)
        deps = [srcp, os.path.join(ROOT, "include", "lsb.h")] + [os.path.join(CSRC, h) for h in os.listdir(CSRC)
                                                                  if h.endswith(".cuh")]
        if not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(d) for d in deps):
            cmd = [NVCC, *ARCH, *COMMON, *dflags, *EXTRA.get(src, []), "-c", srcp, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
        objs.append(obj)
    cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
