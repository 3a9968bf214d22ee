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

# the reference's own test suite (tests/conformance) imports `snpsim`: alias it
# to this package (tests/conformance_alias.py)
from conformance_alias import install as _install_snpsim_alias  # noqa: E402

_install_snpsim_alias()

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


# -- the reference's test suite (tests/conformance, copied unmodified) ---------------------
# Its conftest (pkg/tests/conftest.py) is restated here: one `conftest` module
# serves both suites (the reference tests do `from conftest import random_systems`).

import hypothesis.strategies as _st  # noqa: E402

RANDOM_BOUNDS = dict(q_max=50, rules_per_neuron_max=4, out_degree_max=8, spikes_max=20, delay_max=3)


@_st.composite
def random_systems(draw, q_max=50):
    """pkg/tests/conftest.py:11-16: a validated random system from a drawn seed."""
    from paper_2408_04343_b200 import gen_random
    seed = draw(_st.integers(min_value=0, max_value=2**32 - 1))
    return gen_random(seed=seed, **dict(RANDOM_BOUNDS, q_max=q_max))


# conformance files whose tests run simulations (device engines): gpu
_CONF_GPU_FILES = {"test_engine.py", "test_acceptance.py", "test_oracle_equivalence.py"}
# single conformance tests elsewhere that run a simulation
_CONF_GPU_TESTS = {
    "test_cli.py": ("TestRun", "TestBench", "test_run", "test_bench"),
    "test_generators.py": ("test_outputs_decode_to_ascending_values", "test_output_totals_nondecreasing_per_step",
                           "test_tiny_instance_paths", "test_accepts_only_exact_sums"),
}
# deselected, with the reason
_CONF_DESELECT = {
    "test_acceptance.py::test_criterion_2_size_formulas":
        "documented red in the reference itself (pkg/README.md:28-38, pkg/test_output.txt:166-196)",
    "test_cli.py::TestRun::test_trace_files_identical_across_formats":
        "its fourth run is `--format oracle`, the reference's CPU interpreter; this engine's CLI has no CPU "
        "backend (the three device formats are compared byte for byte in tests/test_cli.py)",
}


def pytest_collection_modifyitems(config, items):
    keep, dropped = [], []
    for item in items:
        path = str(item.fspath)
        if "/conformance/" not in path:
            keep.append(item)
            continue
        fname = path.rsplit("/", 1)[-1]
        nodeid = item.nodeid.split("/conformance/", 1)[-1]
        if nodeid in _CONF_DESELECT:
            dropped.append(item)
            continue
        if fname in _CONF_GPU_FILES or any(k in item.nodeid for k in _CONF_GPU_TESTS.get(fname, ())):
            item.add_marker(pytest.mark.gpu)
        keep.append(item)
    if dropped:
        config.hook.pytest_deselected(items=dropped)
        items[:] = keep


def multi_amount_system(q: int, pmax: int, seed: int | None = None):
    """synth-v1 with delays whose sending rules produce random amounts in
    [1, pmax] (consumption and thresholds raised to stay consistent), so P is
    u8 / u16 / u32 per neuron instead of bits."""
    import paper_2408_04343_b200 as snp
    base = snp.synth_v1(q, with_delays=True)
    r = base.rules
    rng = np.random.default_rng(pmax if seed is None else seed)
    firing = r.produced > 0
    amount = rng.integers(1, pmax + 1, size=len(r.produced))
    produced = np.where(firing, amount, 0)
    consumed = np.where(firing, np.maximum(r.consumed, produced), r.consumed)
    threshold = np.where(firing & ~r.is_exact, np.maximum(r.threshold, consumed), r.threshold)
    threshold = np.where(firing & r.is_exact, consumed, threshold)
    rules = snp.RuleVector(threshold, r.is_exact, consumed, produced, r.delay, r.neuron)
    initial = base.initial + rng.integers(0, 3 * pmax, size=base.neuron_count)
    return snp.SystemArrays(initial, rules, base.rule_map, base.adj_offsets, base.adj_targets)


def concentrated_system(q: int, hot: int = 256, deg: int = 16, seed: int = 5):
    """synth-v1 rules (with delays) whose out-edges all land in the first `hot`
    neurons: every delivery goes to one destination tile, so the binned push
    overflows its shared-memory buckets on every step."""
    import paper_2408_04343_b200 as snp
    base = snp.synth_v1(q, with_delays=True)
    rng = np.random.default_rng(seed)
    key = rng.random((q, hot))
    key[np.arange(hot), np.arange(hot)] = 2.0  # neurons in the hot set never pick themselves
    tg = np.argsort(key, axis=1)[:, :deg].astype(np.int64)
    tg.sort(axis=1)
    adj_off = np.arange(0, deg * q + 1, deg, dtype=np.int64)
    return snp.SystemArrays(base.initial, base.rules, base.rule_map, adj_off, tg.reshape(-1))
