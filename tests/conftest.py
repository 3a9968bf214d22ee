"""Shared fixtures.  `-m gpu` tests need a B200 (run through gpurun);
everything else runs on CPU.  The golden fixtures under tests/golden were
produced by the reference itself (tests/golden/make_golden.py)."""

from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

ORACLE_FIELDS = ("initial", "offsets", "threshold", "is_exact", "consumed", "produced", "delay",
                 "adj_offsets", "adj_targets")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; run via gpurun")


@lru_cache(maxsize=None)
def golden_npz(name: str):
    return dict(np.load(GOLDEN / name, allow_pickle=False))


@lru_cache(maxsize=None)
def golden_json(name: str):
    return json.loads((GOLDEN / name).read_text())


def corpus_system(i: int):
    """System ``i`` of the C3 corpus as an oracle.OracleSystem."""
    from oracle.snp_oracle import OracleSystem
    c = golden_npz("corpus.npz")
    parts = {}
    for f in ORACLE_FIELDS:
        idx = c[f + "__idx"]
        parts[f] = c[f][idx[i]:idx[i + 1]]
    return OracleSystem.from_npz(parts)


def corpus_size() -> int:
    return len(golden_npz("corpus.npz")["digest_first"])


def scenario_names() -> list[str]:
    t = golden_npz("traces.npz")
    return sorted({k.split("/")[0] for k in t if "/sys/" in k})


def scenario_system(name: str):
    from oracle.snp_oracle import OracleSystem
    t = golden_npz("traces.npz")
    return OracleSystem.from_npz(t, prefix=f"{name}/sys/")


def scenario_trace(name: str, tag: str) -> dict:
    t = golden_npz("traces.npz")
    pre = f"{name}/{tag}/"
    return {k[len(pre):]: t[k] for k in t if k.startswith(pre)}


def to_system_arrays(osys):
    """OracleSystem -> product SystemArrays (plain data conversion)."""
    from paper_2408_04343_b200.generators import SystemArrays
    from paper_2408_04343_b200.matrices import NeuronRuleMap, RuleVector
    owner = np.repeat(np.arange(osys.q, dtype=np.int64), np.diff(osys.offsets))
    rules = RuleVector(osys.threshold.copy(), osys.is_exact.copy(), osys.consumed.copy(),
                       osys.produced.copy(), osys.delay.copy(), owner)
    return SystemArrays(osys.initial.copy(), rules, NeuronRuleMap(osys.offsets.copy()),
                        osys.adj_offsets.copy(), osys.adj_targets.copy())


@pytest.fixture
def empty_system():
    from paper_2408_04343_b200 import SNPSystem
    return SNPSystem().validate()
