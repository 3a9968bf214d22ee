"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and
records its outputs; the fixtures are committed so that the oracle
restatement (oracle/) and the B200 engine are pinned to the reference even
on the GPU box, where /root/reference does not exist.

Fixtures (all produced by reference calls, file:line of the reference API):
* tables.json      -- Tables 1-3 for sort n=3: build_sparse/build_ell/
                      build_compressed (matrices.py:143-187), rule offsets
                      (matrices.py:134-137)
* mix64_kat.json   -- selection.mix64 (selection.py:37-45) known answers
* traces.npz       -- FULL traces (simulate, engine.py:405-461) of the sort
                      family (n=3,5,10), the delay scenarios of
                      test_engine.py / test_acceptance.py, subset-sum (1,2)/3
* corpus.npz       -- 1000 gen_random(50,4,8,20,3,seed) systems (the C3
                      acceptance corpus, test_acceptance.py:151-167) as arrays
                      plus sha256 digests of their FULL traces (L=100) under
                      FirstApplicable and SeededRandom(seed)
* synth.npz        -- synth-v1 systems (q=1000, with/without delays) run
                      through the reference simulate_prepared via the
                      direct-array Prepared shim, 12 steps,
                      both policies: full traces
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import snpsim  # noqa: E402  (the reference)
from snpsim import engine as ref_engine  # noqa: E402
from snpsim.matrices import (NeuronRuleMap as RNeuronRuleMap, RuleVector as RRuleVector,  # noqa: E402
                             SynapseMatrix as RSynapseMatrix)

from oracle.snp_oracle import trace_digest  # noqa: E402


def ref_arrays(system) -> dict:
    """Reference rule vector + sorted out-neighbours as flat arrays."""
    rules, rule_map = snpsim.build_rule_vector(system)
    q = system.neuron_count
    off = np.zeros(q + 1, dtype=np.int64)
    dst = []
    for i in range(q):
        nb = system.out_neighbors(i)
        off[i + 1] = off[i] + len(nb)
        dst.extend(nb)
    return {
        "initial": np.asarray(system.initial_spikes, dtype=np.int64),
        "offsets": rule_map.offsets.astype(np.int64),
        "threshold": rules.threshold, "is_exact": rules.is_exact, "consumed": rules.consumed,
        "produced": rules.produced, "delay": rules.delay,
        "adj_offsets": off, "adj_targets": np.asarray(dst, dtype=np.int64),
    }


def trace_arrays(trace) -> dict:
    out = {"configs": np.stack(trace.configs).astype(np.int64),
           "halt": np.array(trace.halt_reason.value)}
    if trace.delays is not None:
        out["delays"] = np.stack(trace.delays).astype(np.int64)
    if trace.spiking is not None:
        q = trace.configs[0].shape[0]
        out["spiking"] = (np.stack(trace.spiking).astype(np.int64) if trace.spiking
                          else np.zeros((0, q), dtype=np.int64))
    return out


def tables():
    system = snpsim.gen_sort(snpsim.SortInstance(3))
    sp = snpsim.build_sparse(system)
    ell = snpsim.build_ell(system)
    syn = snpsim.build_compressed(system)
    _, rm = snpsim.build_rule_vector(system)
    doc = {
        "sparse": sp.data.tolist(),
        "ell_target": ell.target.tolist(), "ell_amount": ell.amount.tolist(),
        "compressed": syn.target.tolist(),
        "offsets": rm.offsets.tolist(),
        "storage": {f"sort100/{f.value}": snpsim.storage_elements(f, snpsim.gen_sort(snpsim.SortInstance(100)))
                    for f in snpsim.matrices.MATRIX_FORMATS},
    }
    (HERE / "tables.json").write_text(json.dumps(doc, indent=1))


def mix_kat():
    from snpsim.selection import mix64
    seeds = [0, 1, 12345, 2**63, 2**64 - 1, 240804343]
    steps = [0, 1, 7, 10**6]
    neurons = [0, 1, 10**7 - 1, 10**8 - 1]
    rows = [[s, k, n, mix64(s, k, n)] for s in seeds for k in steps for n in neurons]
    (HERE / "mix64_kat.json").write_text(json.dumps(rows))


def scenario_systems():
    S = snpsim
    out = {}

    def relay(c=2, p=1, d=0, init=(2, 0)):
        s = S.SNPSystem()
        a = s.add_neuron(init[0])
        b = s.add_neuron(init[1])
        s.add_rule(a, S.at_least(c), c, p, d)
        s.add_synapse(a, b)
        return s.validate()

    out["relay"] = relay()
    # test_engine.py:298-309 / test_acceptance.py:219-231: fires at [0, 3, 6]
    s = S.SNPSystem()
    a, b = s.add_neuron(3), s.add_neuron(0)
    s.add_rule(a, S.at_least(1), 1, 1, 2)
    s.add_synapse(a, b)
    out["delay_close"] = s.validate()
    # test_acceptance.py:233-252: lost spikes into a closed neuron
    s = S.SNPSystem()
    src, dst = s.add_neuron(3), s.add_neuron(1)
    s.add_rule(src, S.at_least(1), 1, 1, 0)
    s.add_rule(dst, S.at_least(1), 1, 1, 2)
    s.add_synapse(src, dst)
    out["lost_spikes"] = s.validate()
    # test_engine.py:311-321: spin-free reopening
    s = S.SNPSystem()
    a = s.add_neuron(1)
    s.add_rule(a, S.at_least(1), 1, 1, 3)
    out["spin_free"] = s.validate()
    # test_engine.py:176-189: forgetting only subtracts
    s = S.SNPSystem()
    a, b = s.add_neuron(3), s.add_neuron(0)
    s.add_rule(a, S.exactly(3), 3, 0, 0)
    s.add_synapse(a, b)
    out["forgetting"] = s.validate()
    # test_engine.py:191-212: padding
    s = S.SNPSystem()
    for _ in range(4):
        s.add_neuron(0)
    s.add_neuron(1)
    for d in (1, 2, 3):
        s.add_synapse(0, d)
    s.add_rule(4, S.at_least(1), 1, 1, 0)
    s.add_synapse(4, 1)
    out["padding"] = s.validate()
    # test_engine.py:214-224: zero rows (no synapses)
    s = S.SNPSystem()
    s.add_neuron(1)
    s.add_rule(0, S.at_least(1), 1, 1, 0)
    out["zero_rows"] = s.validate()
    # test_engine.py:273-280: no rules -> immediate halt
    s = S.SNPSystem()
    s.add_neuron(5)
    out["no_rules"] = s.validate()
    # first-applicable prefers the lower index (test_engine.py:86-95)
    s = S.SNPSystem()
    a = s.add_neuron(2)
    s.add_rule(a, S.exactly(2), 2, 1, 0)
    s.add_rule(a, S.at_least(1), 1, 1, 0)
    out["two_rules"] = s.validate()
    out["sort3"] = S.gen_sort(S.SortInstance(3))
    out["sort5"] = S.gen_sort(S.SortInstance(5))
    out["sort10"] = S.gen_sort(S.SortInstance(10))
    out["sort10_random_values"] = S.gen_sort(S.SortInstance(10, (7, 3, 19, 1, 12, 5, 30, 2, 8, 11)))
    out["subset12"] = S.gen_subset_sum(S.SubsetSumInstance((1, 2), 3))
    out["subset_rand8"] = S.gen_subset_sum(S.SubsetSumInstance.random(8, seed=8))
    return out


def traces():
    S = snpsim
    data = {}
    for name, system in scenario_systems().items():
        for k, v in ref_arrays(system).items():
            data[f"{name}/sys/{k}"] = v
        runs = [("first", S.FirstApplicable(), 60), ("seeded7", S.SeededRandom(7), 60),
                ("seeded_big", S.SeededRandom(2**63 + 5), 60)]
        for tag, sel, L in runs:
            opts = S.SimOptions(max_steps=L, selection=sel, record=S.RecordLevel.FULL)
            tr = S.simulate(system, S.Format.ORACLE, opts)
            for k, v in trace_arrays(tr).items():
                data[f"{name}/{tag}/{k}"] = v
    # subset-sum acceptance over 200 seeds (test_acceptance.py:186-216)
    sys12 = scenario_systems()["subset12"]
    acc = []
    for seed in range(200):
        tr = S.simulate(sys12, S.Format.COMPRESSED,
                        S.SimOptions(max_steps=S.generators.SUBSET_SUM_STEP_BOUND,
                                     selection=S.SeededRandom(seed)))
        acc.append(int(tr.configs[-1][sys12.output_neuron]))
    data["subset12/accept_final_adder"] = np.asarray(acc, dtype=np.int64)
    # sort n=100: CONFIGS digest and decode (test_acceptance.py:170-183)
    s100 = S.gen_sort(S.SortInstance(100))
    tr = S.simulate(s100, S.Format.COMPRESSED, S.SimOptions(max_steps=110))
    data["sort100/digest"] = np.array(trace_digest(tr.configs))
    data["sort100/final"] = tr.configs[-1]
    data["sort100/steps"] = np.array(tr.steps)
    np.savez_compressed(HERE / "traces.npz", **data)


def corpus(n_systems: int = 1000, L: int = 100):
    S = snpsim
    fields = ("initial", "offsets", "threshold", "is_exact", "consumed", "produced", "delay",
              "adj_offsets", "adj_targets")
    cat = {f: [] for f in fields}
    idx = {f: [0] for f in fields}
    dig_first, dig_seeded, halt_first, halt_seeded, steps_first, steps_seeded = [], [], [], [], [], []
    t0 = time.time()
    for seed in range(n_systems):
        system = S.gen_random(50, 4, 8, 20, 3, seed)
        arr = ref_arrays(system)
        for f in fields:
            cat[f].append(np.asarray(arr[f]))
            idx[f].append(idx[f][-1] + len(arr[f]))
        for sel, dl, hl, sl in ((S.FirstApplicable(), dig_first, halt_first, steps_first),
                                (S.SeededRandom(seed), dig_seeded, halt_seeded, steps_seeded)):
            tr = S.simulate(system, S.Format.COMPRESSED,
                            S.SimOptions(max_steps=L, selection=sel, record=S.RecordLevel.FULL))
            dl.append(trace_digest(tr.configs, tr.delays, tr.spiking))
            hl.append(tr.halt_reason.value)
            sl.append(tr.steps)
    out = {}
    for f in fields:
        out[f] = np.concatenate(cat[f]).astype(np.int32 if f != "is_exact" else bool)
        out[f + "__idx"] = np.asarray(idx[f], dtype=np.int64)
    out["digest_first"] = np.asarray(dig_first)
    out["digest_seeded"] = np.asarray(dig_seeded)
    out["halt_first"] = np.asarray(halt_first)
    out["halt_seeded"] = np.asarray(halt_seeded)
    out["steps_first"] = np.asarray(steps_first)
    out["steps_seeded"] = np.asarray(steps_seeded)
    out["L"] = np.array(L)
    np.savez_compressed(HERE / "corpus.npz", **out)
    print(f"corpus: {n_systems} systems in {time.time() - t0:.1f}s")


class _Shim:
    """The only system fields simulate_prepared reads (engine.py:427-428)."""

    def __init__(self, initial):
        self.initial_spikes = initial
        self.neuron_count = len(initial)


def synth(steps: int = 12):
    from paper_2408_04343_b200.generators import synth_v1  # pure numpy, no device needed
    S = snpsim
    data = {}
    for tag, q, delays in (("k3", 1000, False), ("k4", 1000, True), ("k3big", 20000, False)):
        a = synth_v1(q, with_delays=delays)
        r = a.rules
        rv = RRuleVector(r.threshold.copy(), r.is_exact.copy(), r.consumed.copy(), r.produced.copy(),
                         r.delay.copy(), r.neuron.copy())
        rm = RNeuronRuleMap(a.rule_map.offsets.copy())
        z = 16
        syn = np.full((z, q), -1, dtype=np.int64)
        syn[np.tile(np.arange(z), q), np.repeat(np.arange(q), z)] = a.adj_targets
        prep = ref_engine.Prepared(_Shim(a.initial.copy()), S.Format.COMPRESSED, rv, rm, RSynapseMatrix(syn))
        for pol, sel in (("first", S.FirstApplicable()), ("seeded", S.SeededRandom(99))):
            tr = S.simulate_prepared(prep, S.SimOptions(max_steps=steps, selection=sel,
                                                       record=S.RecordLevel.FULL))
            if q <= 1000:
                for k, v in trace_arrays(tr).items():
                    data[f"{tag}/{pol}/{k}"] = v
            else:
                data[f"{tag}/{pol}/digest"] = np.array(trace_digest(tr.configs, tr.delays, tr.spiking))
                data[f"{tag}/{pol}/final"] = tr.configs[-1]
        data[f"{tag}/q"] = np.array(q)
        data[f"{tag}/delays"] = np.array(delays)
    data["steps"] = np.array(steps)
    np.savez_compressed(HERE / "synth.npz", **data)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tables", "mix", "traces", "corpus", "synth"]
    if "tables" in which:
        tables()
    if "mix" in which:
        mix_kat()
    if "traces" in which:
        traces()
    if "corpus" in which:
        corpus()
    if "synth" in which:
        synth()
    print("golden fixtures written to", HERE)
