"""Build libsnpb200.so in-tree with nvcc for sm_100a (no JIT, no torch
extension): ``python -m paper_2408_04343_b200.build``.

The engine is compiled as several objects in parallel: snp_engine.cu (host
runtime + every non-tiled kernel) and snp_tiled.cu once per P mode (the
tiled kernel's instances), then linked into one shared library."""

from __future__ import annotations

import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
HEADERS = [CSRC / "snp_device.cuh", CSRC / "snp_ingest.cuh", PKG.parent / "include" / "snpb200.h"]
OUT = PKG / "libsnpb200.so"
OBJ_DIR = PKG / "build_obj"
CU_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
            "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills"]
# (object name, source, extra defines)
UNITS = [("snp_engine", CSRC / "snp_engine.cu", [])] + [
    (f"snp_tiled_pm{pm}", CSRC / "snp_tiled.cu", [f"-DSNP_TILED_PM={pm}"]) for pm in range(4)]
SOURCES = [CSRC / "snp_engine.cu", CSRC / "snp_tiled.cu"]
DEPS = SOURCES + HEADERS
# kept for tools that compile the engine in one nvcc call
NVCC_FLAGS = CU_FLAGS + ["-shared"]

IO_SOURCES = [CSRC / "snp_modelio.cpp"]
IO_DEPS = IO_SOURCES + [PKG.parent / "include" / "snpio.h"]
IO_OUT = PKG / "libsnpio.so"
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-Wextra"]


def _stale(out: Path, deps: list[Path]) -> bool:
    return not out.exists() or any(out.stat().st_mtime < d.stat().st_mtime for d in deps)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Build libsnpb200.so (nvcc, sm_100a) and libsnpio.so (g++, host-only
    model-file I/O)."""
    if force or _stale(OUT, DEPS):
        OBJ_DIR.mkdir(exist_ok=True)
        jobs = []
        for name, src, defs in UNITS:
            obj = OBJ_DIR / f"{name}.o"
            if force or _stale(obj, [src] + HEADERS):
                jobs.append(["nvcc", *CU_FLAGS, *defs, "-c", "-o", str(obj), str(src)])
        with ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
            for f in [ex.submit(_run, cmd, verbose) for cmd in jobs]:
                f.result()
        _run(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(OUT),
              *[str(OBJ_DIR / f"{name}.o") for name, _, _ in UNITS]], verbose)
    if force or _stale(IO_OUT, IO_DEPS):
        _run(["g++", *CXX_FLAGS, "-o", str(IO_OUT), *map(str, IO_SOURCES)], verbose)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
