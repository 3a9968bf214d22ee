"""bench.py's reference arm: the unmodified reference (baseline/_ref) driven
through the direct-array shim on the bench workload (CPU)."""

import numpy as np
import pytest

import bench
import paper_2408_04343_b200 as snp
from oracle import coracle
from oracle.snp_oracle import OracleSystem

snpsim = bench.import_reference()
needs_ref = pytest.mark.skipif(snpsim is None, reason="reference not installed in baseline/_ref")


@needs_ref
@pytest.mark.parametrize("delays", [False, True])
def test_reference_synth_is_synth_v1(delays):
    q = 5000
    init, rv, rm, syn = bench.reference_synth(snpsim, q, delays)
    a = snp.generators.synth_v1_numpy(q, with_delays=delays)
    np.testing.assert_array_equal(init, a.initial)
    for f in ("threshold", "is_exact", "consumed", "produced", "delay", "neuron"):
        np.testing.assert_array_equal(getattr(rv, f), getattr(a.rules, f))
    np.testing.assert_array_equal(rm.offsets, a.rule_map.offsets)
    np.testing.assert_array_equal(syn.target.T.reshape(-1), a.adj_targets)


@needs_ref
def test_reference_arm_runs_the_reference_engine():
    """The shimmed Prepared through snpsim.simulate_prepared == the C oracle."""
    ref_engine = snpsim.engine
    q, steps = 3000, 6
    init, rv, rm, syn = bench.reference_synth(snpsim, q, True)
    prep = ref_engine.Prepared(bench._Shim(init), snpsim.Format.COMPRESSED, rv, rm, syn)
    tr = snpsim.simulate_prepared(prep, snpsim.SimOptions(max_steps=steps, selection=snpsim.SeededRandom(240804343),
                                                          workers=4))
    _, want, _ = coracle.run(OracleSystem.from_arrays(snp.synth_v1(q, with_delays=True)), steps, 1, 240804343)
    np.testing.assert_array_equal(tr.configs[-1], want)
    assert snpsim.__file__.startswith(str(bench.REF_DIR))


def test_host_info_fields():
    h = bench.host_info()
    assert h["numpy"] == np.__version__ and h["logical_cpus"] >= 1
