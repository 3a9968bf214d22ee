"""Run one degenerate system on one format/variant (debug tool; a hang is caught by the caller's timeout).
    python tools/debug_edge.py FMT VARIANT CASE RECORD"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2408_04343_b200 as snp  # noqa: E402

fmt, variant, case, rec = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
s = snp.SNPSystem()
if case == 1:
    s.add_neuron(5)
elif case == 2:
    a = s.add_neuron(2)
    s.add_rule(a, snp.exactly(3), 1, 1, 0)
elif case == 3:
    x, y = s.add_neuron(1), s.add_neuron(0)
    s.add_rule(x, snp.at_least(1), 1, 1, 0)
    s.add_rule(y, snp.at_least(1), 1, 1, 0)
    s.add_synapse(x, y)
    s.add_synapse(y, x)
s.validate()
tr = snp.simulate_prepared(snp.prepare(s, snp.Format(fmt), variant=variant),
                           snp.SimOptions(max_steps=4, record=snp.RecordLevel[rec]))
print("ok", fmt, variant, case, rec, tr.halt_reason, [c.tolist() for c in tr.configs], flush=True)
