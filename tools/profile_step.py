"""Run a few SNP steps of a workload (for ncu captures; numbers printed here
are not bench values)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2408_04343_b200 as snp  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--workload", default="k3")
p.add_argument("--format", default="compressed")
p.add_argument("--variant", default="tiled")
p.add_argument("--policy", default="first")
p.add_argument("--steps", type=int, default=6)
p.add_argument("--q", type=int, default=10_000_000)
p.add_argument("--sort", type=int, default=0, help="sort instance n (workload ignored)")
a = p.parse_args()
if a.sort:
    arrays = snp.sort_arrays(snp.SortInstance(a.sort))
elif a.workload == "k2":
    arrays = snp.sort_arrays(snp.SortInstance(4096))
else:
    arrays = snp.synth_v1(a.q, with_delays=a.workload == "k4")
prep = snp.prepare(arrays, snp.Format(a.format), variant=a.variant if a.format == "compressed" else "auto")
sel = snp.FirstApplicable() if a.policy == "first" else snp.SeededRandom(240804343)
prep.engine.begin()
tot, kms, _ = prep.engine.time_steps(a.steps, sel, per_kernel=True)
info = prep.engine.info
print(f"{a.workload}/{a.format}/{a.variant}/{a.policy}: {tot / a.steps:.3f} ms/step, step kernel {kms:.3f} ms "
      f"tile={info['tile']} n_tiles={info['n_tiles']} ring={info.get('ring_stages')}x{info.get('stage_bytes')} acc{info.get('counter_bits')} words={info['in_edges']} dev_MB={info['device_bytes'] >> 20}")
