"""Host-side API: builder/validation (model.py), the reference interchange
layouts (matrices.py) against the reference's Tables 1-3, storage
accounting, and the workload generators.  CPU only."""

from collections import Counter

import numpy as np
import pytest

import paper_2408_04343_b200 as snp
from conftest import corpus_size, corpus_system, golden_json
from paper_2408_04343_b200.matrices import NULL, adjacency_from_synapse_matrix


# -- Tables 1-3 (test_acceptance.py:50-122) ---------------------------------------------

def test_tables_match_reference():
    t = golden_json("tables.json")
    system = snp.gen_sort(snp.SortInstance(3))
    assert snp.build_sparse(system).data.tolist() == t["sparse"]
    ell = snp.build_ell(system)
    assert ell.target.tolist() == t["ell_target"]
    assert ell.amount.tolist() == t["ell_amount"]
    assert snp.build_compressed(system).target.tolist() == t["compressed"]
    _, rm = snp.build_rule_vector(system)
    assert rm.offsets.tolist() == t["offsets"] == [0, 1, 2, 3, 6, 9, 12, 12, 12, 12]


def test_storage_formulas_match_reference():
    t = golden_json("tables.json")["storage"]
    system = snp.gen_sort(snp.SortInstance(100))
    for fmt in snp.MATRIX_FORMATS:
        assert snp.storage_elements(fmt, system) == t[f"sort100/{fmt.value}"]
    assert snp.storage_elements(snp.Format.COMPRESSED, system) == 71_301
    with pytest.raises(ValueError):
        snp.storage_elements(snp.Format.ORACLE, system)
    q = system.neuron_count
    for fmt in snp.MATRIX_FORMATS:
        assert snp.storage_bytes(fmt, system) == (snp.storage_elements(fmt, system) - q) * 4 + q * 8


def test_empty_system_layouts(empty_system):
    for fmt in snp.MATRIX_FORMATS:
        assert snp.storage_elements(fmt, empty_system) == 1
    rules, rm = snp.build_rule_vector(empty_system)
    assert len(rules) == 0 and rm.offsets.tolist() == [0]
    assert snp.build_compressed(empty_system).target.shape == (0, 0)


def test_no_synapses_zero_rows_and_one_ell_row():
    s = snp.SNPSystem()
    s.add_neuron(2)
    s.add_rule(0, snp.at_least(1), 1, 1, 0)
    s.validate()
    assert snp.build_compressed(s).rows == 0
    ell = snp.build_ell(s)
    assert ell.rows == 1 and ell.target[0, 0] == 0 and ell.amount[0, 0] == -1


# -- corpus: the C3 systems, independent reconstructions -------------------------------------

def _reconstruct_dense(system):
    rows = []
    for rule in system.rules:
        row = [0] * system.neuron_count
        row[rule.neuron] = -rule.consumed
        if rule.produced:
            for src, dst in system.synapses:
                if src == rule.neuron:
                    row[dst] = rule.produced
        rows.append(row)
    return rows


@pytest.mark.parametrize("seed", list(range(0, 1000, 37)))
def test_gen_random_reproduces_reference_corpus(seed):
    """Same random.Random call order as generators.py:195-230 -> same systems."""
    system = snp.gen_random(50, 4, 8, 20, 3, seed)
    a = snp.system_arrays(system)
    gold = corpus_system(seed)
    np.testing.assert_array_equal(a.initial, gold.initial)
    np.testing.assert_array_equal(a.rule_map.offsets, gold.offsets)
    for f in ("threshold", "is_exact", "consumed", "produced", "delay"):
        np.testing.assert_array_equal(getattr(a.rules, f), getattr(gold, f))
    np.testing.assert_array_equal(a.adj_offsets, gold.adj_offsets)
    np.testing.assert_array_equal(a.adj_targets, gold.adj_targets)
    # layouts agree with independent reconstructions (test_matrices.py:31-165)
    assert snp.build_sparse(system).data.tolist() == _reconstruct_dense(system)
    ell = snp.build_ell(system)
    syn = snp.build_compressed(system)
    for ri, rule in enumerate(system.rules):
        col = [(int(ell.target[r, ri]), int(ell.amount[r, ri])) for r in range(ell.rows)
               if ell.target[r, ri] != NULL]
        assert col[0] == (rule.neuron, -rule.consumed)
        want = [(d, rule.produced) for d in system.out_neighbors(rule.neuron)] if rule.produced else []
        assert col[1:] == want
    for n in range(system.neuron_count):
        col = [int(v) for v in syn.target[:, n] if v != NULL]
        assert col == system.out_neighbors(n)
    off, dst = adjacency_from_synapse_matrix(syn)
    np.testing.assert_array_equal(off, a.adj_offsets)
    np.testing.assert_array_equal(dst, a.adj_targets)


def test_corpus_size():
    assert corpus_size() == 1000


def test_offsets_and_grouping():
    for seed in range(20):
        system = snp.gen_random(50, 4, 8, 20, 3, seed)
        rules, rm = snp.build_rule_vector(system)
        per = Counter(r.neuron for r in system.rules)
        assert np.diff(rm.offsets).tolist() == [per.get(i, 0) for i in range(system.neuron_count)]
        assert list(rules.neuron) == sorted(rules.neuron)


# -- model invariants (model.py:40-112, test_model.py) -----------------------------------------

def test_regex_and_rule_invariants():
    assert snp.at_least(0).matches(0) and snp.at_least(2).matches(5) and not snp.at_least(2).matches(1)
    assert snp.exactly(3).matches(3) and not snp.exactly(3).matches(4)
    with pytest.raises(snp.InvalidRule):
        snp.exactly(0)
    with pytest.raises(snp.InvalidRule):
        snp.at_least(-1)
    with pytest.raises(snp.InvalidRule):
        snp.Rule(0, snp.at_least(1), 1, 2, 0)
    with pytest.raises(snp.InvalidRule):
        snp.Rule(0, snp.exactly(2), 2, 0, 1)
    with pytest.raises(snp.InvalidRule):
        snp.Rule(0, snp.at_least(2), 2, 0, 0)
    with pytest.raises(snp.InvalidRule):
        snp.Rule(0, snp.at_least(1), 0, 0, 0)
    assert snp.Rule(0, snp.exactly(2), 2, 0, 0).is_forgetting


def test_builder_errors_and_stable_regroup():
    s = snp.SNPSystem()
    a, b = s.add_neuron(0), s.add_neuron(0)
    with pytest.raises(snp.ReflexiveSynapse):
        s.add_synapse(a, a)
    with pytest.raises(snp.UnknownNeuron):
        s.add_synapse(a, 7)
    with pytest.raises(snp.UnknownNeuron):
        s.add_rule(5, snp.at_least(1), 1, 1)
    with pytest.raises(snp.ModelError):
        s.add_neuron(-1)
    s.add_rule(b, snp.at_least(1), 1, 1)
    s.add_rule(a, snp.at_least(2), 2, 1)
    s.add_rule(b, snp.at_least(3), 3, 1)
    s.add_synapse(a, b)
    s.add_synapse(a, b)
    s.validate()
    assert [r.neuron for r in s.rules] == [0, 1, 1]
    assert [r.regex.threshold for r in s.rules] == [2, 1, 3]  # per-neuron order kept
    assert s.synapses == {(0, 1)}
    assert s.stats() == snp.SystemStats(2, 3, 1, 2, 1)


# -- array generators --------------------------------------------------------------------------

@pytest.mark.parametrize("n", [1, 2, 3, 7, 40])
def test_sort_arrays_equal_builder(n):
    a = snp.sort_arrays(snp.SortInstance(n))
    b = snp.system_arrays(snp.gen_sort(snp.SortInstance(n)))
    np.testing.assert_array_equal(a.initial, b.initial)
    np.testing.assert_array_equal(a.rule_map.offsets, b.rule_map.offsets)
    for f in ("threshold", "is_exact", "consumed", "produced", "delay", "neuron"):
        np.testing.assert_array_equal(getattr(a.rules, f), getattr(b.rules, f))
    np.testing.assert_array_equal(a.adj_offsets, b.adj_offsets)
    np.testing.assert_array_equal(a.adj_targets, b.adj_targets)


@pytest.mark.parametrize("q,delays", [(17, False), (1000, True), (123457, False)])
def test_synth_v1_shape(q, delays):
    a = snp.synth_v1(q, with_delays=delays)
    assert a.rule_count == 4 * q
    deg = np.diff(a.adj_offsets)
    assert (deg == 16).all()
    t = a.adj_targets.reshape(q, 16)
    assert (np.diff(t, axis=1) > 0).all()            # ascending and distinct
    assert (t != np.arange(q)[:, None]).all()          # non-reflexive
    assert ((t >= 0) & (t < q)).all()
    # rule invariants of model.py:72-112 hold for every generated rule
    r = a.rules
    forget = r.produced == 0
    assert (r.is_exact[forget]).all() and (r.threshold[forget] == r.consumed[forget]).all()
    assert (r.delay[forget] == 0).all()
    assert (r.consumed[~forget] >= r.produced[~forget]).all() and (r.produced[~forget] >= 1).all()
    assert (r.delay.max() <= 3) and (delays or r.delay.max() == 0)


def test_format_aliases():
    assert snp.Format.OPTIMIZED is snp.Format.COMPRESSED
    assert snp.Format.DENSE is snp.Format.SPARSE
    assert [f.value for f in snp.Format] == ["sparse", "ell", "compressed", "oracle"]
    with pytest.raises(ValueError):
        snp.Format("dense")


def test_oracle_format_is_not_a_product_backend():
    with pytest.raises(ValueError, match="oracle"):
        snp.prepare(snp.gen_sort(snp.SortInstance(3)), snp.Format.ORACLE)


def test_sim_options_validation():
    with pytest.raises(ValueError):
        snp.SimOptions(max_steps=0)
    with pytest.raises(ValueError):
        snp.SimOptions(max_steps=1, workers=0)


def test_selection_hash_vector_matches_scalar():
    from paper_2408_04343_b200.selection import choose_index, mix64, mix64_array
    neurons = np.arange(97)
    for seed in (0, 1, 12345, 2**63):
        for step in (0, 7):
            v = mix64_array(seed, step, neurons)
            assert [int(x) for x in v] == [mix64(seed, step, int(n)) for n in neurons]
    for seed in range(50):
        assert 0 <= choose_index(snp.SeededRandom(seed), 3, 5, 4) < 4
    assert choose_index(snp.FirstApplicable(), 0, 0, 9) == 0
    kat = golden_json("mix64_kat.json")
    assert all(mix64(s, k, n) == w for s, k, n, w in kat)


def test_phase_cache_key_handles_empty_arrays():
    """Zero-size inputs (e.g. a 0-row SynapseMatrix) still get a content key."""
    from paper_2408_04343_b200.engine import _content_key
    assert _content_key(np.zeros((0, 3), np.int64)) != _content_key(np.zeros((3, 0), np.int64))
    assert _content_key(np.zeros(0, np.int64), np.arange(3)) == _content_key(np.zeros(0, np.int64), np.arange(3))
