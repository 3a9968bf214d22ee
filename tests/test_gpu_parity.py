"""B200 engine vs the reference (golden fixtures) and the pinned CPU oracle.

Every test here runs the CUDA kernels through the C ABI (libsnpb200.so) and
requires bit-exact equality: configurations, delays, spiking vectors (global
rule ids) and halting step/reason at every step.
"""

import numpy as np
import pytest

import paper_2408_04343_b200 as snp
from conftest import (corpus_size, corpus_system, golden_npz, scenario_names, scenario_system,
                      scenario_trace, to_system_arrays)
from oracle import coracle
from oracle.snp_oracle import OracleSystem, trace_digest

pytestmark = pytest.mark.gpu

FORMATS = [(snp.Format.SPARSE, "auto"), (snp.Format.ELL, "auto"), (snp.Format.COMPRESSED, "tiled"),
           (snp.Format.COMPRESSED, "pull"), (snp.Format.COMPRESSED, "push"), (snp.Format.COMPRESSED, "small")]
FMT_IDS = ["sparse", "ell", "compressed-tiled", "compressed-pull", "compressed-push", "compressed-small"]
POLICIES = {"first": snp.FirstApplicable(), "seeded7": snp.SeededRandom(7),
            "seeded_big": snp.SeededRandom(2**63 + 5)}


def _check(trace, gold):
    assert trace.halt_reason.value == str(gold["halt"])
    np.testing.assert_array_equal(np.stack(trace.configs), gold["configs"])
    if "delays" in gold:
        np.testing.assert_array_equal(np.stack(trace.delays), gold["delays"])
    if "spiking" in gold:
        q = gold["configs"].shape[1]
        sp = np.stack(trace.spiking) if trace.spiking else np.zeros((0, q), np.int64)
        np.testing.assert_array_equal(sp, gold["spiking"])


# -- whole-run traces vs the reference ----------------------------------------------------

@pytest.mark.parametrize("fmt,variant", FORMATS, ids=FMT_IDS)
@pytest.mark.parametrize("name", scenario_names())
def test_scenarios_match_reference(fmt, variant, name):
    prep = snp.prepare(to_system_arrays(scenario_system(name)), fmt, variant=variant)
    for tag, sel in POLICIES.items():
        tr = snp.simulate_prepared(prep, snp.SimOptions(max_steps=60, selection=sel,
                                                        record=snp.RecordLevel.FULL))
        _check(tr, scenario_trace(name, tag))


@pytest.mark.parametrize("fmt,variant", FORMATS, ids=FMT_IDS)
def test_corpus_matches_reference_digests(fmt, variant):
    """C3 (test_acceptance.py:151-167): 1000 random systems x 2 policies,
    L=100, FULL traces identical to the reference (sha256 of every row)."""
    c = golden_npz("corpus.npz")
    L = int(c["L"])
    n = corpus_size() if (fmt is snp.Format.COMPRESSED and variant == "tiled") else 400
    for i in range(n):
        prep = snp.prepare(to_system_arrays(corpus_system(i)), fmt, variant=variant)
        for sel, key in ((snp.FirstApplicable(), "first"), (snp.SeededRandom(i), "seeded")):
            tr = snp.simulate_prepared(prep, snp.SimOptions(max_steps=L, selection=sel,
                                                            record=snp.RecordLevel.FULL))
            assert trace_digest(tr.configs, tr.delays, tr.spiking) == c[f"digest_{key}"][i], (i, key)


@pytest.mark.parametrize("tag", ["k3", "k4"])
@pytest.mark.parametrize("fmt,variant", FORMATS, ids=FMT_IDS)
def test_synth_matches_reference(tag, fmt, variant):
    d = golden_npz("synth.npz")
    a = snp.synth_v1(int(d[f"{tag}/q"]), with_delays=bool(d[f"{tag}/delays"]))
    prep = snp.prepare(a, fmt, variant=variant)
    for pol, sel in (("first", snp.FirstApplicable()), ("seeded", snp.SeededRandom(99))):
        gold = {k.split("/")[-1]: d[k] for k in d if k.startswith(f"{tag}/{pol}/")}
        tr = snp.simulate_prepared(prep, snp.SimOptions(max_steps=int(d["steps"]), selection=sel,
                                                        record=snp.RecordLevel.FULL))
        _check(tr, gold)


def test_synth_20k_digest():
    d = golden_npz("synth.npz")
    prep = snp.prepare(snp.synth_v1(int(d["k3big/q"])), snp.Format.COMPRESSED)
    for pol, sel in (("first", snp.FirstApplicable()), ("seeded", snp.SeededRandom(99))):
        tr = snp.simulate_prepared(prep, snp.SimOptions(max_steps=int(d["steps"]), selection=sel,
                                                        record=snp.RecordLevel.FULL))
        assert trace_digest(tr.configs, tr.delays, tr.spiking) == str(d[f"k3big/{pol}/digest"])


# -- sort family (test_acceptance.py:170-183; section 6) -------------------------

@pytest.mark.parametrize("fmt,variant", FORMATS, ids=FMT_IDS)
@pytest.mark.parametrize("n", [3, 5, 10, 100])
def test_sorting_end_to_end(fmt, variant, n):
    prep = snp.prepare(snp.gen_sort(snp.SortInstance(n)), fmt, variant=variant)
    tr = snp.simulate_prepared(prep, snp.SimOptions(max_steps=n + 10))
    assert tr.halt_reason is snp.HaltReason.NO_APPLICABLE_RULES
    assert snp.sort_result(tr, n) == list(range(1, n + 1))
    if n == 100:
        t = golden_npz("traces.npz")
        assert trace_digest(tr.configs) == str(t["sort100/digest"])


@pytest.mark.parametrize("n,fmts", [(512, FORMATS), (2048, [(snp.Format.COMPRESSED, "tiled"),
                                                            (snp.Format.COMPRESSED, "pull"),
                                                            (snp.Format.COMPRESSED, "push")])])
def test_sort_large_halts_sorted(n, fmts):
    """Heavy-neuron path (detectors own n rules and n in-neighbours)."""
    rng = np.random.default_rng(n)
    values = tuple(int(v) for v in rng.choice(np.arange(1, 4 * n), size=n, replace=False))
    a = snp.sort_arrays(snp.SortInstance(n, values))
    want_final = None
    for fmt, variant in fmts:
        prep = snp.prepare(a, fmt, variant=variant)
        res = snp.run_final(prep, snp.SimOptions(max_steps=5 * n))
        assert res.halt_reason is snp.HaltReason.NO_APPLICABLE_RULES
        assert res.config[2 * n:].tolist() == sorted(values)
        if want_final is None:
            want_final = res.config
        np.testing.assert_array_equal(res.config, want_final)
    # the first 40 steps are bit-exact against the C oracle
    tr, _, _ = coracle.run(OracleSystem.from_arrays(a), 40, trace_rows=41)
    prep = snp.prepare(a, snp.Format.COMPRESSED)
    mine = snp.simulate_prepared(prep, snp.SimOptions(max_steps=40, record=snp.RecordLevel.FULL))
    assert trace_digest(mine.configs, mine.delays, mine.spiking) == trace_digest(tr.configs, tr.delays, tr.spiking)


@pytest.mark.parametrize("variant", ["tiled", "pull"])
@pytest.mark.parametrize("policy", ["first", "seeded"])
def test_k2_sort4096_to_halt(variant, policy):
    """K2 (BASELINE.json configs[1]): the worst-case sorter n=4096 (values
    n..1) runs n+1 = 4097 steps to NO_APPLICABLE_RULES and decodes 1..n
    (test_acceptance.py:170-183); the first 50 FULL trace rows equal the C
    oracle's (oracle.py:21-101)."""
    n = 4096
    a = snp.sort_arrays(snp.SortInstance(n))
    sel, pol, seed = ((snp.FirstApplicable(), 0, 0) if policy == "first"
                      else (snp.SeededRandom(240804343), 1, 240804343))
    prep = snp.prepare(a, snp.Format.COMPRESSED, variant=variant)
    res = snp.run_final(prep, snp.SimOptions(max_steps=n + 10, selection=sel))
    assert res.halt_reason is snp.HaltReason.NO_APPLICABLE_RULES
    assert res.steps == n + 1
    assert res.config[2 * n:].tolist() == list(range(1, n + 1))
    ref, _, _ = coracle.run(OracleSystem.from_arrays(a), 50, pol, seed, trace_rows=51)
    mine = snp.simulate_prepared(prep, snp.SimOptions(max_steps=50, selection=sel, record=snp.RecordLevel.FULL))
    assert trace_digest(mine.configs, mine.delays, mine.spiking) == trace_digest(ref.configs, ref.delays, ref.spiking)


@pytest.mark.parametrize("fmt", [snp.Format.ELL, snp.Format.SPARSE], ids=["ell", "sparse"])
def test_sort2048_ell_sparse_to_halt(fmt):
    """ELL (69 GB of pairs) and the dense matrix (103 GB) at sort n=2048:
    run to halt, decode, and match the oracle's first 30 FULL rows."""
    n = 2048
    rng = np.random.default_rng(7)
    values = tuple(int(v) for v in rng.choice(np.arange(1, 4 * n), size=n, replace=False))
    a = snp.sort_arrays(snp.SortInstance(n, values))
    prep = snp.prepare(a, fmt)
    res = snp.run_final(prep, snp.SimOptions(max_steps=5 * n))
    assert res.halt_reason is snp.HaltReason.NO_APPLICABLE_RULES
    assert res.config[2 * n:].tolist() == sorted(values)
    full, want_c, _ = coracle.run(OracleSystem.from_arrays(a), 5 * n, 0, 0)
    assert res.steps == full.n_steps
    np.testing.assert_array_equal(res.config, want_c)
    # a 30-step run has 31 config rows but 30 spiking rows
    ref, _, _ = coracle.run(OracleSystem.from_arrays(a), 30, 0, 0, trace_rows=31)
    mine = snp.simulate_prepared(prep, snp.SimOptions(max_steps=30, record=snp.RecordLevel.FULL))
    assert trace_digest(mine.configs, mine.delays, mine.spiking) == trace_digest(ref.configs, ref.delays, ref.spiking)
    del prep


def test_subset_sum_accepting_paths():
    t = golden_npz("traces.npz")
    prep = snp.prepare(to_system_arrays(scenario_system("subset12")), snp.Format.COMPRESSED)
    adder = scenario_system("subset12").q - 1
    got = [int(snp.run_final(prep, snp.SimOptions(max_steps=6, selection=snp.SeededRandom(s))).config[adder])
           for s in range(200)]
    assert got == t["subset12/accept_final_adder"].tolist()
    assert 0 in got  # some seed accepts


# -- full-size parity (K3 / K4 at 10^7 against the C oracle) ------------------------------

@pytest.mark.parametrize("delays,policy", [(False, 0), (True, 1)])
def test_full_size_synth_steps_bit_exact(delays, policy):
    q, steps = 10_000_000, 3
    a = snp.synth_v1(q, with_delays=delays)
    sel = snp.FirstApplicable() if policy == 0 else snp.SeededRandom(240804343)
    seed = 0 if policy == 0 else 240804343
    prep = snp.prepare(a, snp.Format.COMPRESSED)
    res = snp.run_final(prep, snp.SimOptions(max_steps=steps, selection=sel))
    _, want_c, want_d = coracle.run(OracleSystem.from_arrays(a), steps, policy, seed)
    np.testing.assert_array_equal(res.config, want_c)
    np.testing.assert_array_equal(res.delays, want_d)
    assert res.steps == steps and res.halt_reason is snp.HaltReason.STEP_LIMIT


@pytest.mark.parametrize("delays,policy", [(False, 0), (True, 0), (False, 1), (True, 1)])
def test_lean_kernel_many_steps_bit_exact(delays, policy):
    """Unrecorded runs take the lean tiled instance (no trace / counters, fast
    phase-2 selection); 60 steps of it must equal the C oracle and the final
    row of a recorded (non-lean) run."""
    q, steps = 300_000, 60
    a = snp.synth_v1(q, with_delays=delays)
    sel = snp.FirstApplicable() if policy == 0 else snp.SeededRandom(2**63 + 5)
    seed = 0 if policy == 0 else 2**63 + 5
    prep = snp.prepare(a, snp.Format.COMPRESSED)
    res = snp.run_final(prep, snp.SimOptions(max_steps=steps, selection=sel))
    _, want_c, want_d = coracle.run(OracleSystem.from_arrays(a), steps, policy, seed)
    np.testing.assert_array_equal(res.config, want_c)
    np.testing.assert_array_equal(res.delays, want_d)
    tr = snp.simulate_prepared(prep, snp.SimOptions(max_steps=steps, selection=sel,
                                                    record=snp.RecordLevel.CONFIGS_AND_DELAYS))
    np.testing.assert_array_equal(tr.configs[-1], want_c)
    np.testing.assert_array_equal(tr.delays[-1], want_d)


@pytest.mark.parametrize("tag", ["k3", "k4"])
def test_full_size_formats_match_oracle(tag):
    """K3 / K4 at 10^7: every COMPRESSED variant and ELL, 4 steps under
    FirstApplicable and SeededRandom, equal the C oracle (configuration and
    delays)."""
    q, steps = 10_000_000, 4
    a = snp.synth_v1(q, with_delays=tag == "k4")
    osys = OracleSystem.from_arrays(a)
    want = {pol: coracle.run(osys, steps, pol, 240804343)[1:] for pol in (0, 1)}
    for fmt, variant in [(snp.Format.COMPRESSED, "tiled"), (snp.Format.COMPRESSED, "pull"),
                         (snp.Format.COMPRESSED, "push"), (snp.Format.ELL, "auto")]:
        prep = snp.prepare(a, fmt, variant=variant)
        for pol, sel in ((0, snp.FirstApplicable()), (1, snp.SeededRandom(240804343))):
            res = snp.run_final(prep, snp.SimOptions(max_steps=steps, selection=sel))
            assert res.steps == steps and res.halt_reason is snp.HaltReason.STEP_LIMIT
            np.testing.assert_array_equal(res.config, want[pol][0], err_msg=f"{fmt} {variant} {pol}")
            np.testing.assert_array_equal(res.delays, want[pol][1], err_msg=f"{fmt} {variant} {pol}")
        del prep


# -- phase functions (test_engine.py:66-259) --------------------------------------------------

def _relay(c=2, p=1, d=0):
    s = snp.SNPSystem()
    a, b = s.add_neuron(2), s.add_neuron(0)
    s.add_rule(a, snp.at_least(c), c, p, d)
    s.add_synapse(a, b)
    return s.validate()


def test_sv_calc_sorter_detector():
    system = snp.gen_sort(snp.SortInstance(3))
    rules, rm = snp.build_rule_vector(system)
    cfg = np.zeros(9, dtype=np.int64)
    cfg[3] = 3
    sv = snp.sv_calc(cfg, np.zeros(9, dtype=np.int64), rules, rm, snp.FirstApplicable())
    assert sv.chosen[3] == 3 and sv.flags(12).sum() == 1


def test_sv_calc_closed_and_first_applicable():
    system = _relay()
    rules, rm = snp.build_rule_vector(system)
    sv = snp.sv_calc(np.array([2, 0]), np.array([1, 2]), rules, rm, snp.FirstApplicable())
    assert sv.is_empty
    s = snp.SNPSystem()
    a = s.add_neuron(2)
    s.add_rule(a, snp.exactly(2), 2, 1, 0)
    s.add_rule(a, snp.at_least(1), 1, 1, 0)
    s.validate()
    rules, rm = snp.build_rule_vector(s)
    assert snp.sv_calc(np.array([2]), np.zeros(1, np.int64), rules, rm, snp.FirstApplicable()).chosen[0] == 0
    # seeded: roughly uniform over seeds (test_engine.py:97-111), exactly the reference's picks
    from paper_2408_04343_b200.selection import mix64
    first = 0
    for seed in range(2000):
        ch = snp.sv_calc(np.array([2]), np.zeros(1, np.int64), rules, rm, snp.SeededRandom(seed)).chosen[0]
        assert ch == mix64(seed, 0, 0) % 2
        first += ch == 0
    assert abs(first / 2000 - 0.5) <= 0.05


def test_sv_calc_matches_oracle_with_random_state():
    from oracle.snp_oracle import VectorEngine
    rng = np.random.default_rng(5)
    for i in range(0, 1000, 97):
        osys = corpus_system(i)
        a = to_system_arrays(osys)
        ve = VectorEngine(osys, "compressed")
        for trial in range(3):
            cfg = rng.integers(0, 21, osys.q)
            dly = rng.integers(0, 3, osys.q) * (rng.random(osys.q) < 0.3)
            for pol, seed in ((0, 0), (1, 1234 + trial)):
                sel = snp.FirstApplicable() if pol == 0 else snp.SeededRandom(seed)
                got = snp.sv_calc(cfg, dly, a.rules, a.rule_map, sel, step=trial * 11).chosen
                np.testing.assert_array_equal(got, ve.sv_calc(cfg, dly, pol, seed, trial * 11))


def test_step_kernels_match_oracle_with_random_state():
    from oracle.snp_oracle import VectorEngine
    rng = np.random.default_rng(9)
    for i in range(0, 1000, 89):
        osys = corpus_system(i)
        system = snp.gen_random(50, 4, 8, 20, 3, i)
        rules, rm = snp.build_rule_vector(system)
        mats = {"sparse": snp.build_sparse(system), "ell": snp.build_ell(system),
                "compressed": snp.build_compressed(system)}
        for trial in range(3):
            cfg = rng.integers(0, 21, osys.q) + 40  # large enough to never go negative
            dly = rng.integers(0, 3, osys.q) * (rng.random(osys.q) < 0.3)
            chosen = VectorEngine(osys, "compressed").sv_calc(cfg, dly * 0, 0, 0, 0)
            state = snp.SimState(cfg, dly, snp.SpikingVector(chosen))
            for fmt, fn in (("sparse", snp.step_sparse), ("ell", snp.step_ell), ("compressed", snp.step_compressed)):
                want = VectorEngine(osys, fmt).step(cfg, dly, chosen)
                np.testing.assert_array_equal(fn(state, mats[fmt], rules), want)
            want_d = VectorEngine(osys, "compressed").update_delays(dly, chosen)
            np.testing.assert_array_equal(snp.update_delays(dly, snp.SpikingVector(chosen), rules), want_d)


def test_step_single_rule_identity_and_closed_destination():
    system = _relay()
    rules, rm = snp.build_rule_vector(system)
    mats = (snp.build_sparse(system), snp.build_ell(system), snp.build_compressed(system))
    fns = (snp.step_sparse, snp.step_ell, snp.step_compressed)
    cfg, z = np.array([2, 0]), np.zeros(2, dtype=np.int64)
    sv = snp.sv_calc(cfg, z, rules, rm, snp.FirstApplicable())
    for fn, mat in zip(fns, mats):
        assert fn(snp.SimState(cfg, z, sv), mat, rules).tolist() == [0, 1]
        empty = snp.SimState(np.array([1, 5]), z, snp.SpikingVector(np.full(2, -1, dtype=np.int64)))
        assert fn(empty, mat, rules).tolist() == [1, 5]
        closed = snp.SimState(np.array([2, 7]), np.array([0, 3]), sv)
        assert fn(closed, mat, rules).tolist() == [0, 7]


def test_ell_row_visits():
    system = snp.gen_sort(snp.SortInstance(3))
    rules, rm = snp.build_rule_vector(system)
    cfg = np.zeros(9, dtype=np.int64)
    cfg[3] = 2
    z = np.zeros(9, dtype=np.int64)
    sv = snp.sv_calc(cfg, z, rules, rm, snp.FirstApplicable())
    visits = np.zeros(12, dtype=np.int64)
    snp.step_ell(snp.SimState(cfg, z, sv), snp.build_ell(system), rules, row_visits=visits)
    assert visits[int(sv.chosen[3])] == 2


def test_update_delays_cases():
    s = snp.SNPSystem()
    a = s.add_neuron(1)
    s.add_rule(a, snp.at_least(1), 1, 1, 3)
    rules = snp.build_rule_vector(s.validate())[0]
    none = snp.SpikingVector(np.full(3, -1, dtype=np.int64))
    assert snp.update_delays(np.array([0, 2, 1]), none, rules).tolist() == [0, 1, 0]
    assert snp.update_delays(np.zeros(1, np.int64), snp.SpikingVector(np.array([0])), rules).tolist() == [3]


def test_negative_spikes_every_format():
    s = snp.SNPSystem()
    a = s.add_neuron(1)
    s.add_rule(a, snp.at_least(1), 2, 1, 0)
    s.validate()
    for fmt, variant in FORMATS:
        with pytest.raises(snp.NegativeSpikes):
            snp.simulate(s, fmt, snp.SimOptions(max_steps=5)) if variant == "auto" else \
                snp.simulate_prepared(snp.prepare(s, fmt, variant=variant), snp.SimOptions(max_steps=5))


def test_loop_contract():
    system = snp.gen_sort(snp.SortInstance(3))
    tr = snp.simulate(system, snp.Format.SPARSE, snp.SimOptions(max_steps=1))
    assert len(tr.configs) == 2 and tr.halt_reason is snp.HaltReason.STEP_LIMIT
    s = snp.SNPSystem()
    s.add_neuron(5)
    s.validate()
    tr = snp.simulate(s, snp.Format.COMPRESSED, snp.SimOptions(max_steps=10))
    assert tr.halt_reason is snp.HaltReason.NO_APPLICABLE_RULES and [c.tolist() for c in tr.configs] == [[5]]
    empty = snp.SNPSystem().validate()
    tr = snp.simulate(empty, snp.Format.SPARSE, snp.SimOptions(max_steps=3))
    assert tr.halt_reason is snp.HaltReason.NO_APPLICABLE_RULES and len(tr.configs) == 1
    lean = snp.simulate(system, snp.Format.ELL, snp.SimOptions(max_steps=10))
    assert lean.delays is None and lean.spiking is None
    full = snp.simulate(system, snp.Format.ELL, snp.SimOptions(max_steps=10, record=snp.RecordLevel.FULL))
    assert len(full.spiking) == full.steps and len(full.delays) == len(full.configs)
    assert snp.format_trace(snp.simulate(_relay(), snp.Format.SPARSE, snp.SimOptions(max_steps=5))).splitlines()[0] == "2 0"


def test_trace_chunking_is_invisible():
    """Long recorded runs cross several device segments and host copies."""
    a = snp.sort_arrays(snp.SortInstance(300))
    prep = snp.prepare(a, snp.Format.COMPRESSED)
    opts = snp.SimOptions(max_steps=400, record=snp.RecordLevel.FULL)
    t1 = prep.engine.trace(opts, rows_per_call=7)
    t2 = prep.engine.trace(opts)
    assert t1 == t2 and t1.halt_reason is snp.HaltReason.NO_APPLICABLE_RULES
    assert t1.configs[-1][600:].tolist() == list(range(1, 301))


# -- device trace digests (SNP_REC_DIGEST) ------------------------------------------------

@pytest.mark.parametrize("policy", ["first", "seeded7"])
def test_trace_digests_match_rows(policy):
    """Digests computed on the device equal row_digest of the recorded rows
    (full trace of the same run) and of the C oracle's rows."""
    a = snp.synth_v1(30_000, with_delays=True)
    sel = POLICIES[policy]
    prep = snp.prepare(a, snp.Format.COMPRESSED)
    opts = snp.SimOptions(max_steps=25, selection=sel, record=snp.RecordLevel.FULL)
    tr = snp.simulate_prepared(prep, opts)
    dg = snp.trace_digests(prep, opts)
    assert dg.halt_reason is tr.halt_reason and dg.steps == tr.steps
    assert [int(x) for x in dg.configs] == [snp.row_digest(r) for r in tr.configs]
    assert [int(x) for x in dg.delays] == [snp.row_digest(r) for r in tr.delays]
    assert [int(x) for x in dg.spiking] == [snp.row_digest(r) for r in tr.spiking]
    seed = 0 if policy == "first" else 7
    ref, _, _ = coracle.run(OracleSystem.from_arrays(a), 25, 0 if policy == "first" else 1, seed, trace_rows=26)
    assert [int(x) for x in dg.configs] == [snp.row_digest(r) for r in ref.configs]


def test_trace_digests_sorter_halts():
    a = snp.sort_arrays(snp.SortInstance(50))
    for fmt, var in [(snp.Format.COMPRESSED, "tiled"), (snp.Format.ELL, "auto")]:
        prep = snp.prepare(a, fmt, variant=var)
        opts = snp.SimOptions(max_steps=200, record=snp.RecordLevel.CONFIGS)
        dg = snp.trace_digests(prep, opts)
        tr = snp.simulate_prepared(prep, opts)
        assert dg.halt_reason is snp.HaltReason.NO_APPLICABLE_RULES and dg.steps == tr.steps
        assert [int(x) for x in dg.configs] == [snp.row_digest(r) for r in tr.configs]
        assert dg.delays is None and dg.spiking is None


# -- device-side ingest: the tiled layout built on the GPU == the host reference build ----------

def _sparse_far_system(q=400_000, edges=50_000, seed=5):
    """Few edges between far-apart neurons: segments cut by the 2^17 source-span rule."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, q, edges)
    dst = rng.integers(0, q, edges)
    keep = src != dst
    pairs = np.unique(np.stack([src[keep], dst[keep]], axis=1), axis=0)
    off = np.zeros(q + 1, np.int64)
    np.cumsum(np.bincount(pairs[:, 0], minlength=q), out=off[1:])
    base = snp.synth_v1(q)
    return snp.SystemArrays(base.initial, base.rules, base.rule_map, off, pairs[:, 1].astype(np.int64))


@pytest.mark.parametrize("case", ["synth", "synth_delays", "sort300", "sparse_far", "tiny"])
def test_device_layout_build_matches_host(case, monkeypatch):
    if case == "synth":
        a = snp.synth_v1(700_000)
    elif case == "synth_delays":
        a = snp.synth_v1(123_457, with_delays=True)
    elif case == "sort300":
        a = snp.sort_arrays(snp.SortInstance(300))
    elif case == "sparse_far":
        a = _sparse_far_system()
    else:
        a = snp.synth_v1(17)
    digests = []
    finals = []
    for dev in ("0", "1"):
        monkeypatch.setenv("SNPB200_DEVICE_BUILD", dev)
        prep = snp.prepare(a, snp.Format.COMPRESSED, variant="tiled")
        digests.append(prep.engine.layout_digest())
        finals.append(snp.run_final(prep, snp.SimOptions(max_steps=8, selection=snp.SeededRandom(4))).config)
        del prep
    assert digests[0] == digests[1]
    assert any(digests[0])
    np.testing.assert_array_equal(finals[0], finals[1])


# -- two-pass receive (variant tiled2) -------------------------------------------------------

@pytest.mark.parametrize("case", ["synth", "synth_delays_seeded", "sort300", "sparse_far"])
def test_tiled2_matches_oracle(case):
    if case == "sort300":
        a, L, sel, pol, seed = snp.sort_arrays(snp.SortInstance(300)), 310, snp.FirstApplicable(), 0, 0
    elif case == "sparse_far":
        a, L, sel, pol, seed = _sparse_far_system(), 20, snp.SeededRandom(3), 1, 3
    else:
        d = case != "synth"
        a = snp.synth_v1(250_000, with_delays=d)
        L, sel, pol, seed = 30, (snp.SeededRandom(9) if d else snp.FirstApplicable()), (1 if d else 0), (9 if d else 0)
    prep = snp.prepare(a, snp.Format.COMPRESSED, variant="tiled2")
    res = snp.run_final(prep, snp.SimOptions(max_steps=L, selection=sel))
    _, want_c, want_d = coracle.run(OracleSystem.from_arrays(a), L, pol, seed)
    np.testing.assert_array_equal(res.config, want_c)
    np.testing.assert_array_equal(res.delays, want_d)
    tr = snp.simulate_prepared(prep, snp.SimOptions(max_steps=12, selection=sel, record=snp.RecordLevel.FULL))
    ref, _, _ = coracle.run(OracleSystem.from_arrays(a), 12, pol, seed, trace_rows=13)
    assert trace_digest(tr.configs, tr.delays, tr.spiking) == trace_digest(ref.configs, ref.delays, ref.spiking)


@pytest.mark.parametrize("name", scenario_names())
def test_tiled2_scenarios(name):
    prep = snp.prepare(to_system_arrays(scenario_system(name)), snp.Format.COMPRESSED, variant="tiled2")
    for tag, sel in POLICIES.items():
        tr = snp.simulate_prepared(prep, snp.SimOptions(max_steps=60, selection=sel, record=snp.RecordLevel.FULL))
        _check(tr, scenario_trace(name, tag))


# -- counts beyond 2^31 (the lean guard compares a saturated 32-bit count) ----------------

@pytest.mark.parametrize("fmt,variant", FORMATS + [(snp.Format.COMPRESSED, "tiled2")],
                         ids=FMT_IDS + ["compressed-tiled2"])
def test_huge_counts_guards(fmt, variant):
    """Spike counts above 2^31 against thresholds near 2^31: exactly-guards
    must not match, at-least guards must, and counts keep growing in int64."""
    big = 2**31 + 5
    s = snp.SNPSystem()
    a = s.add_neuron(big)                       # never equals 2^31-1, is >= 2^31-1
    b = s.add_neuron(2**31 - 1)                 # exactly 2^31-1 at step 0
    c = s.add_neuron(3 * 2**31)                 # far above every threshold
    d = s.add_neuron(0)
    s.add_rule(a, snp.exactly(2**31 - 1), 2**31 - 1, 1, 0)
    s.add_rule(a, snp.at_least(2**31 - 1), 3, 2, 1)
    s.add_rule(b, snp.exactly(2**31 - 1), 2**31 - 1, 5, 0)
    s.add_rule(b, snp.at_least(1), 1, 1, 0)
    s.add_rule(c, snp.at_least(2**30), 2**30, 1, 2)
    s.add_rule(d, snp.at_least(1), 1, 1, 0)
    for x, y in [(a, d), (b, d), (c, d), (d, a), (c, a)]:
        s.add_synapse(x, y)
    s.validate()
    arrays = snp.system_arrays(s)
    prep = snp.prepare(arrays, fmt, variant=variant)
    for pol, seed in ((0, 0), (1, 13)):
        sel = snp.FirstApplicable() if pol == 0 else snp.SeededRandom(seed)
        tr = snp.simulate_prepared(prep, snp.SimOptions(max_steps=12, selection=sel, record=snp.RecordLevel.FULL))
        ref, _, _ = coracle.run(OracleSystem.from_arrays(arrays), 12, pol, seed, trace_rows=13)
        assert trace_digest(tr.configs, tr.delays, tr.spiking) == trace_digest(ref.configs, ref.delays, ref.spiking)
        fin = snp.run_final(prep, snp.SimOptions(max_steps=12, selection=sel))  # lean instance
        np.testing.assert_array_equal(fin.config, np.asarray(tr.configs[-1]))


@pytest.mark.parametrize("pmax", [3, 300, 70_000])
def test_multi_amount_production_paths(pmax):
    """Produced amounts that differ between rules (P as u8 / u16 / u32 per
    neuron instead of bits): tiled (global P lookups), CSR pull and push vs
    the C oracle at 120k neurons."""
    base = snp.synth_v1(120_000, with_delays=True)
    r = base.rules
    rng = np.random.default_rng(pmax)
    firing = r.produced > 0
    amount = rng.integers(1, pmax + 1, size=len(r.produced))
    produced = np.where(firing, amount, 0)
    consumed = np.where(firing, np.maximum(r.consumed, produced), r.consumed)
    threshold = np.where(firing & ~r.is_exact, np.maximum(r.threshold, consumed), r.threshold)
    threshold = np.where(firing & r.is_exact, consumed, threshold)
    rules = snp.RuleVector(threshold, r.is_exact, consumed, produced, r.delay, r.neuron)
    initial = base.initial + rng.integers(0, 3 * pmax, size=base.neuron_count)
    a = snp.SystemArrays(initial, rules, base.rule_map, base.adj_offsets, base.adj_targets)
    _, want_c, want_d = coracle.run(OracleSystem.from_arrays(a), 15, 1, 21)
    for variant in ("tiled", "pull", "push"):
        prep = snp.prepare(a, snp.Format.COMPRESSED, variant=variant)
        res = snp.run_final(prep, snp.SimOptions(max_steps=15, selection=snp.SeededRandom(21)))
        np.testing.assert_array_equal(res.config, want_c, err_msg=variant)
        np.testing.assert_array_equal(res.delays, want_d, err_msg=variant)


@pytest.mark.parametrize("mode", ["binned", "atomic", "unfused"])
@pytest.mark.parametrize("pmax", [1, 300])
def test_push_step_kernels_match_oracle(mode, pmax, monkeypatch):
    """The three ways a push-format run steps (include/snpb200.h SNP_PUSH_*):
    binned deliveries (u16 slots for a common amount, u32 slot|amount
    otherwise), L2 atomics, and the unfused step + scatter kernels -- ELL and
    COMPRESSED-push, with delays, SeededRandom, vs the C oracle: 20 steps of
    final state and 8 FULL trace rows."""
    from conftest import multi_amount_system
    if mode != "binned":
        monkeypatch.setenv("SNPB200_PUSH", mode)
    q = 200_000
    a = snp.synth_v1(q, with_delays=True) if pmax == 1 else multi_amount_system(q, pmax)
    osys = OracleSystem.from_arrays(a)
    _, want_c, want_d = coracle.run(osys, 20, 1, 21)
    ref, _, _ = coracle.run(osys, 8, 1, 21, trace_rows=9)
    for fmt, var in ((snp.Format.ELL, "auto"), (snp.Format.COMPRESSED, "push")):
        prep = snp.prepare(a, fmt, variant=var)
        assert snp._native.PUSH_KERNELS[prep.engine.info["push_kernel"]] == mode
        res = snp.run_final(prep, snp.SimOptions(max_steps=20, selection=snp.SeededRandom(21)))
        np.testing.assert_array_equal(res.config, want_c, err_msg=f"{fmt} {mode}")
        np.testing.assert_array_equal(res.delays, want_d, err_msg=f"{fmt} {mode}")
        tr = snp.simulate_prepared(prep, snp.SimOptions(max_steps=8, selection=snp.SeededRandom(21),
                                                        record=snp.RecordLevel.FULL))
        assert trace_digest(tr.configs, tr.delays, tr.spiking) == trace_digest(ref.configs, ref.delays, ref.spiking)
        del prep


@pytest.mark.parametrize("fmt,var", [(snp.Format.ELL, "auto"), (snp.Format.COMPRESSED, "push")], ids=["ell", "push"])
def test_binned_push_bucket_overflow(fmt, var):
    """Every delivery into one destination tile (50K sources x 16 targets in
    256 neurons): the binned push's shared-memory buckets overflow into the
    tile's overflow region on every step; 12 steps vs the C oracle."""
    from conftest import concentrated_system
    a = concentrated_system(50_000)
    osys = OracleSystem.from_arrays(a)
    _, want_c, want_d = coracle.run(osys, 12, 1, 4)
    prep = snp.prepare(a, fmt, variant=var)
    assert snp._native.PUSH_KERNELS[prep.engine.info["push_kernel"]] == "binned"
    res = snp.run_final(prep, snp.SimOptions(max_steps=12, selection=snp.SeededRandom(4)))
    np.testing.assert_array_equal(res.config, want_c)
    np.testing.assert_array_equal(res.delays, want_d)


def test_run_with_device_buffers():
    """snp_begin / snp_read_state take device pointers too (unified
    addressing): a torch caller runs from and into CUDA tensors with
    device-to-device copies, bit-identical to the host-buffer run."""
    import torch
    a = snp.synth_v1(30_000, with_delays=True)
    prep = snp.prepare(a, snp.Format.COMPRESSED)
    init = np.asarray(a.initial, dtype=np.int64) + 3
    want = snp.run_final(prep, snp.SimOptions(max_steps=9, selection=snp.SeededRandom(2)))  # system's C_0
    want2 = prep.engine.run_final(9, snp.SeededRandom(2), initial=init)
    d_init = torch.from_numpy(init).cuda()
    d_cfg = torch.empty(a.neuron_count, dtype=torch.int64, device="cuda")
    d_dly = torch.empty_like(d_cfg)
    res = prep.engine.run_device(9, d_init, d_cfg, snp.SeededRandom(2), final_delays=d_dly)
    assert int(res.steps) == want2.steps
    np.testing.assert_array_equal(d_cfg.cpu().numpy(), want2.config)
    np.testing.assert_array_equal(d_dly.cpu().numpy(), want2.delays)
    assert not np.array_equal(want.config, want2.config)  # the initial configuration mattered


@pytest.mark.parametrize("fmt,variant", FORMATS + [(snp.Format.COMPRESSED, "tiled2")],
                         ids=FMT_IDS + ["compressed-tiled2"])
def test_edge_systems_every_variant(fmt, variant):
    """Degenerate inputs the reference accepts (engine.py:416-461): no
    neurons, one neuron without rules, a neuron whose only rule never
    applies, and a two-neuron loop that only stops at the step limit."""
    cases = []
    cases.append((snp.SNPSystem().validate(), 3, snp.HaltReason.NO_APPLICABLE_RULES, [[]]))
    s = snp.SNPSystem()
    s.add_neuron(5)
    cases.append((s.validate(), 10, snp.HaltReason.NO_APPLICABLE_RULES, [[5]]))
    s = snp.SNPSystem()
    a = s.add_neuron(2)
    s.add_rule(a, snp.exactly(3), 1, 1, 0)
    cases.append((s.validate(), 10, snp.HaltReason.NO_APPLICABLE_RULES, [[2]]))
    s = snp.SNPSystem()
    x, y = s.add_neuron(1), s.add_neuron(0)
    s.add_rule(x, snp.at_least(1), 1, 1, 0)
    s.add_rule(y, snp.at_least(1), 1, 1, 0)
    s.add_synapse(x, y)
    s.add_synapse(y, x)
    cases.append((s.validate(), 4, snp.HaltReason.STEP_LIMIT, [[1, 0], [0, 1], [1, 0], [0, 1], [1, 0]]))
    for system, L, halt, configs in cases:
        tr = snp.simulate_prepared(snp.prepare(system, fmt, variant=variant),
                                   snp.SimOptions(max_steps=L, record=snp.RecordLevel.FULL))
        assert tr.halt_reason is halt, (system.neuron_count, tr.halt_reason)
        assert [c.tolist() for c in tr.configs] == configs
        ref = snp.simulate(system, snp.Format.COMPRESSED, snp.SimOptions(max_steps=L, record=snp.RecordLevel.FULL))
        assert trace_digest(tr.configs, tr.delays, tr.spiking) == trace_digest(ref.configs, ref.delays, ref.spiking)
