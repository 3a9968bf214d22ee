"""Pin the CPU oracle restatements (oracle/) to the reference's own outputs.

CPU only.  Every fixture was produced by the unmodified reference
(tests/golden/make_golden.py); this proves the checker before it is used to
judge the B200 engine.
"""

import numpy as np
import pytest

from conftest import (corpus_size, corpus_system, golden_json, golden_npz, scenario_names,
                      scenario_system, scenario_trace)
from oracle import coracle
from oracle.snp_oracle import (OracleNegative, OracleSystem, VectorEngine, interpret, mix64,
                               mix64_vec, trace_digest)

POLICIES = {"first": (0, 0), "seeded7": (1, 7), "seeded_big": (1, 2**63 + 5)}


def _same(trace, gold):
    assert trace.halt == str(gold["halt"])
    np.testing.assert_array_equal(np.stack(trace.configs), gold["configs"])
    if "delays" in gold:
        np.testing.assert_array_equal(np.stack(trace.delays), gold["delays"])
    if "spiking" in gold:
        sp = np.stack(trace.spiking) if trace.spiking else np.zeros((0, gold["configs"].shape[1]), np.int64)
        np.testing.assert_array_equal(sp, gold["spiking"])


def test_mix64_known_answers():
    # selection.py:37-45 values recorded from the reference
    rows = golden_json("mix64_kat.json")
    for seed, step, neuron, want in rows:
        assert mix64(seed, step, neuron) == want
        assert coracle.mix64(seed, step, neuron) == want
        assert int(mix64_vec(seed, step, np.array([neuron]))[0]) == want


@pytest.mark.parametrize("name", scenario_names())
@pytest.mark.parametrize("tag", list(POLICIES))
def test_interpreter_matches_reference_traces(name, tag):
    s = scenario_system(name)
    policy, seed = POLICIES[tag]
    _same(interpret(s, 60, policy, seed, "full"), scenario_trace(name, tag))


@pytest.mark.parametrize("fmt", ["sparse", "ell", "compressed"])
@pytest.mark.parametrize("name", scenario_names())
def test_vector_engine_matches_reference_traces(fmt, name):
    s = scenario_system(name)
    for tag, (policy, seed) in POLICIES.items():
        for workers in (1, 3):
            tr = VectorEngine(s, fmt, workers=workers).run(60, policy, seed, record="full")
            _same(tr, scenario_trace(name, tag))


@pytest.mark.parametrize("name", scenario_names())
def test_c_oracle_matches_reference_traces(name):
    s = scenario_system(name)
    for tag, (policy, seed) in POLICIES.items():
        tr, final, _ = coracle.run(s, 60, policy, seed, trace_rows=61)
        _same(tr, scenario_trace(name, tag))
        np.testing.assert_array_equal(final, scenario_trace(name, tag)["configs"][-1])


def test_corpus_digests_all_oracles():
    """The C3 acceptance corpus (test_acceptance.py:151-167): 1000 systems x
    2 policies, L=100, FULL traces -- C oracle on all, numpy engine on a slice."""
    c = golden_npz("corpus.npz")
    L = int(c["L"])
    for i in range(corpus_size()):
        s = corpus_system(i)
        for policy, seed, key in ((0, 0, "first"), (1, i, "seeded")):
            tr, _, _ = coracle.run(s, L, policy, seed, trace_rows=L + 1)
            assert trace_digest(tr.configs, tr.delays, tr.spiking) == c[f"digest_{key}"][i], (i, key)
            assert tr.halt == c[f"halt_{key}"][i]
            if i < 60:
                vt = VectorEngine(s, ("sparse", "ell", "compressed")[i % 3]).run(L, policy, seed, "full")
                assert trace_digest(vt.configs, vt.delays, vt.spiking) == c[f"digest_{key}"][i]


def test_corpus_interpreter_slice():
    c = golden_npz("corpus.npz")
    L = int(c["L"])
    for i in range(0, corpus_size(), 50):
        s = corpus_system(i)
        tr = interpret(s, L, 1, i, "full")
        assert trace_digest(tr.configs, tr.delays, tr.spiking) == c["digest_seeded"][i]


@pytest.mark.parametrize("tag", ["k3", "k4"])
def test_synth_v1_reference_traces(tag):
    """synth-v1 run by the reference's own simulate_prepared (direct-array shim)."""
    from paper_2408_04343_b200.generators import synth_v1
    d = golden_npz("synth.npz")
    q = int(d[f"{tag}/q"])
    s = OracleSystem.from_arrays(synth_v1(q, with_delays=bool(d[f"{tag}/delays"])))
    steps = int(d["steps"])
    for pol, (policy, seed) in (("first", (0, 0)), ("seeded", (1, 99))):
        gold = {k.split("/")[-1]: d[k] for k in d if k.startswith(f"{tag}/{pol}/")}
        tr, _, _ = coracle.run(s, steps, policy, seed, trace_rows=steps + 1)
        _same(tr, gold)
        vt = VectorEngine(s, "compressed", workers=2).run(steps, policy, seed, "full")
        _same(vt, gold)


def test_synth_v1_large_digest():
    from paper_2408_04343_b200.generators import synth_v1
    d = golden_npz("synth.npz")
    q = int(d["k3big/q"])
    s = OracleSystem.from_arrays(synth_v1(q))
    steps = int(d["steps"])
    for pol, (policy, seed) in (("first", (0, 0)), ("seeded", (1, 99))):
        tr, final, _ = coracle.run(s, steps, policy, seed, trace_rows=steps + 1)
        assert trace_digest(tr.configs, tr.delays, tr.spiking) == str(d[f"k3big/{pol}/digest"])
        np.testing.assert_array_equal(final, d[f"k3big/{pol}/final"])


def test_sort100_and_subset_sum():
    t = golden_npz("traces.npz")
    from paper_2408_04343_b200.generators import SortInstance, sort_arrays
    s = OracleSystem.from_arrays(sort_arrays(SortInstance(100)))
    tr, final, _ = coracle.run(s, 110, trace_rows=111)
    assert trace_digest(tr.configs) == str(t["sort100/digest"])
    assert final[200:300].tolist() == list(range(1, 101))
    s12 = scenario_system("subset12")
    acc = [int(coracle.run(s12, 6, 1, seed)[1][-1]) for seed in range(200)]
    assert acc == t["subset12/accept_final_adder"].tolist()


def test_negative_spikes_raise():
    # test_engine.py:226-234: condition below consumption
    s = OracleSystem(np.array([1]), np.array([0, 1]), np.array([1]), np.array([False]), np.array([2]),
                     np.array([1]), np.array([0]), np.array([0, 0]), np.zeros(0, dtype=np.int64))
    with pytest.raises(OracleNegative):
        interpret(s, 5)
    with pytest.raises(OracleNegative):
        coracle.run(s, 5)
    for fmt in ("sparse", "ell", "compressed"):
        with pytest.raises(OracleNegative):
            VectorEngine(s, fmt).run(5)
