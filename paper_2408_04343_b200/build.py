"""Build libsnpb200.so in-tree with nvcc for sm_100a (no JIT, no torch
extension): ``python -m paper_2408_04343_b200.build``."""

from __future__ import annotations

import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
SOURCES = [PKG / "csrc" / "snp_engine.cu"]
DEPS = SOURCES + [PKG / "csrc" / "snp_device.cuh", PKG.parent / "include" / "snpb200.h"]
OUT = PKG / "libsnpb200.so"
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills"]


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and OUT.exists() and all(OUT.stat().st_mtime >= d.stat().st_mtime for d in DEPS):
        return OUT
    cmd = ["nvcc", *NVCC_FLAGS, "-o", str(OUT), *map(str, SOURCES)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
