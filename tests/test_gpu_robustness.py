"""Input validation and cache/overflow corner cases of the device engine
(advisor findings, round 1).  All of them create device engines: gpu."""

import numpy as np
import pytest

import paper_2408_04343_b200 as snp
from paper_2408_04343_b200.cli import main as cli_main
from oracle import coracle
from oracle.snp_oracle import OracleSystem, trace_digest

pytestmark = pytest.mark.gpu


def _fan_in_system(p: int, sources: int = 3):
    """``sources`` neurons each firing a rule that produces ``p`` into one
    sink: the sink receives sources * p in one step (>= 2^32 for p = 2^31-1)."""
    s = snp.SNPSystem()
    srcs = [s.add_neuron(p) for _ in range(sources)]
    sink = s.add_neuron(0)
    other = s.add_neuron(1)          # a second amount: P is per-neuron, not bits
    for x in srcs:
        s.add_rule(x, snp.at_least(p), p, p, 0)
        s.add_synapse(x, sink)
    s.add_rule(other, snp.at_least(1), 1, 1, 0)
    s.add_synapse(other, sink)
    s.add_rule(sink, snp.at_least(2**31 - 1), 1, 1, 0)
    s.add_synapse(sink, other)
    return snp.system_arrays(s.validate())


def test_receive_beyond_32_bits_uses_64_bit_gather():
    a = _fan_in_system(2**31 - 1)
    ref, _, _ = coracle.run(OracleSystem.from_arrays(a), 6, trace_rows=7)
    want = trace_digest(ref.configs, ref.delays, ref.spiking)
    assert ref.configs[1][3] == 3 * (2**31 - 1) + 1  # more than 32 bits in one step
    for fmt, variant in [(snp.Format.COMPRESSED, "auto"), (snp.Format.COMPRESSED, "pull"),
                         (snp.Format.COMPRESSED, "push"), (snp.Format.ELL, "auto")]:
        prep = snp.prepare(a, fmt, variant=variant)
        tr = snp.simulate_prepared(prep, snp.SimOptions(max_steps=6, record=snp.RecordLevel.FULL))
        assert trace_digest(tr.configs, tr.delays, tr.spiking) == want, (fmt, variant)
    # the tiled kernel's receive counters are 32-bit: refused, not wrapped
    with pytest.raises(MemoryError, match="32-bit receive"):
        snp.prepare(a, snp.Format.COMPRESSED, variant="tiled")


def test_malformed_csr_offsets_rejected():
    base = snp.synth_v1(1000)
    for bad in ("first", "decrease"):
        off = base.adj_offsets.copy()
        if bad == "first":
            off[0] = 3
        else:
            off[500] = off[502] + 1
        a = snp.SystemArrays(base.initial, base.rules, base.rule_map, off, base.adj_targets)
        for variant in ("tiled", "pull"):
            with pytest.raises(ValueError, match="adj_offsets"):
                snp.prepare(a, snp.Format.COMPRESSED, variant=variant)


def test_phase_functions_see_in_place_edits():
    s = snp.SNPSystem()
    a = s.add_neuron(2)
    s.add_rule(a, snp.exactly(2), 2, 1, 0)
    s.add_rule(a, snp.at_least(1), 1, 1, 0)
    s.validate()
    rules, rm = snp.build_rule_vector(s)
    z = np.zeros(1, np.int64)
    assert snp.sv_calc(np.array([2]), z, rules, rm, snp.FirstApplicable()).chosen[0] == 0
    rules.threshold[0] = 5          # the reference recomputes from the current arrays
    assert snp.sv_calc(np.array([2]), z, rules, rm, snp.FirstApplicable()).chosen[0] == 1
    mat = snp.build_compressed(s)
    sv = snp.SpikingVector(np.array([1]))
    st = snp.SimState(np.array([2]), z, sv)
    assert snp.step_compressed(st, mat, rules).tolist() == [1]
    rules.consumed[1] = 2
    assert snp.step_compressed(st, mat, rules).tolist() == [0]
    snp.engine.clear_phase_cache()
    assert not snp.engine._PHASE_CACHE


def test_cli_model_beyond_device_int32_is_a_model_error(tmp_path, capsys):
    s = snp.SNPSystem()
    a = s.add_neuron(1)
    s.add_rule(a, snp.at_least(2**31), 1, 1, 0)  # valid for the reference (int64)
    path = tmp_path / "big.snp"
    snp.save_model(path, s.validate())
    assert cli_main(["run", "--model", str(path), "--format", "compressed", "--steps", "3"]) == 2
    assert "model error" in capsys.readouterr().err


def test_cli_flag_conflicts_checked_before_running(tmp_path, capsys):
    rc = cli_main(["run", "--family", "sort", "-n", "5", "--format", "compressed", "--final-only",
                   "--trace-out", str(tmp_path / "t.txt")])
    assert rc == 1 and not (tmp_path / "t.txt").exists()
