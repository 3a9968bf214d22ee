"""ctypes wrapper of liboracle.so (C restatement of oracle.py:21-101).

TEST INFRASTRUCTURE ONLY: used by tests/ and bench.py's CPU arm as the
checker / baseline, never by the product package.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

from .snp_oracle import HALT_NO_APPLICABLE, HALT_STEP_LIMIT, OracleNegative, OracleSystem, OracleTrace

_HERE = Path(__file__).resolve().parent
_LIB = _HERE / "liboracle.so"
_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB


def load():
    global _lib
    if _lib is None:
        if not _LIB.exists():
            build()
        lib = ctypes.CDLL(str(_LIB))
        vp = ctypes.c_void_p
        lib.oracle_run.restype = ctypes.c_int
        lib.oracle_run.argtypes = [ctypes.c_int64] + [vp] * 9 + [
            ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp]
        lib.oracle_mix64.restype = ctypes.c_uint64
        lib.oracle_mix64.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64]
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def mix64(seed: int, step: int, neuron: int) -> int:
    return int(load().oracle_mix64(seed & ((1 << 64) - 1), step, neuron))


def run(s: OracleSystem, max_steps: int, policy: int = 0, seed: int = 0, trace_rows: int = 0,
        initial: np.ndarray | None = None) -> tuple[OracleTrace, np.ndarray, np.ndarray]:
    """Run to halt; returns (trace of the first ``trace_rows`` rows, final C, final D)."""
    lib = load()
    q = s.q
    c = lambda a: np.ascontiguousarray(a, dtype=np.int64)
    init = c(s.initial if initial is None else initial)
    ex = np.ascontiguousarray(s.is_exact, dtype=np.uint8)
    arrs = [c(s.offsets), c(s.threshold), ex, c(s.consumed), c(s.produced), c(s.delay),
            c(s.adj_offsets), c(s.adj_targets)]
    rows = int(trace_rows)
    tc = np.zeros((rows, q), dtype=np.int64) if rows else None
    td = np.zeros((rows, q), dtype=np.int64) if rows else None
    ts = np.zeros((rows, q), dtype=np.int64) if rows else None
    steps = ctypes.c_int64()
    halt = ctypes.c_int()
    neg = ctypes.c_int64(-1)
    fc = np.empty(q, dtype=np.int64)
    fd = np.empty(q, dtype=np.int64)
    rc = lib.oracle_run(q, _p(init), *[_p(a) for a in arrs], int(max_steps), int(policy),
                        int(seed) & ((1 << 64) - 1), rows, _p(tc), _p(td), _p(ts),
                        ctypes.byref(steps), ctypes.byref(halt), _p(fc), _p(fd), ctypes.byref(neg))
    if rc == 1:
        raise OracleNegative(f"spike count of neuron {neg.value} went negative")
    if rc != 0:
        raise RuntimeError(f"oracle_run failed ({rc})")
    n = steps.value
    nrow = min(rows, n + 1)
    tr = OracleTrace(
        configs=list(tc[:nrow]) if rows else [],
        halt=HALT_STEP_LIMIT if halt.value == 1 else HALT_NO_APPLICABLE,
        delays=list(td[:nrow]) if rows else None,
        spiking=list(ts[:min(rows, n)]) if rows else None)
    tr.n_steps = n
    return tr, fc, fd
