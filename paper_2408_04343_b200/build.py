"""Build libsnpb200.so in-tree with nvcc for sm_100a (no JIT, no torch
extension): ``python -m paper_2408_04343_b200.build``."""

from __future__ import annotations

import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
SOURCES = [PKG / "csrc" / "snp_engine.cu"]
DEPS = SOURCES + [PKG / "csrc" / "snp_device.cuh", PKG / "csrc" / "snp_ingest.cuh", PKG.parent / "include" / "snpb200.h"]
OUT = PKG / "libsnpb200.so"
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills"]


IO_SOURCES = [PKG / "csrc" / "snp_modelio.cpp"]
IO_DEPS = IO_SOURCES + [PKG.parent / "include" / "snpio.h"]
IO_OUT = PKG / "libsnpio.so"
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-Wextra"]


def _stale(out: Path, deps: list[Path]) -> bool:
    return not out.exists() or any(out.stat().st_mtime < d.stat().st_mtime for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Build libsnpb200.so (nvcc, sm_100a) and libsnpio.so (g++, host-only
    model-file I/O)."""
    jobs = []
    if force or _stale(OUT, DEPS):
        jobs.append(["nvcc", *NVCC_FLAGS, "-o", str(OUT), *map(str, SOURCES)])
    if force or _stale(IO_OUT, IO_DEPS):
        jobs.append(["g++", *CXX_FLAGS, "-o", str(IO_OUT), *map(str, IO_SOURCES)])
    for cmd in jobs:
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
