"""Time one rank's step kernel(s) of a row-partitioned system in isolation
(no exchange: the other ranks' P chunks stay zero, which does not change the
work per step).  Numbers printed here are per-rank compute, not bench values.

    python tools/rank_step_time.py --world 8 --rows 10000000 --variant tiled2
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2408_04343_b200 as snp  # noqa: E402
from paper_2408_04343_b200 import sharded as shd  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--world", type=int, default=8)
p.add_argument("--rows", type=int, default=10_000_000)
p.add_argument("--variant", default="tiled")
p.add_argument("--steps", type=int, default=30)
a = p.parse_args()
q = a.rows * a.world
L = shd.shard_layout(q, a.world)
lo, hi = L.bounds(0)
t0 = time.perf_counter()
local = shd.synth_v1_rows(q, lo, hi)
t1 = time.perf_counter()
sh = shd.ShardedEngine(local, q, 0, a.world, variant=a.variant)
t2 = time.perf_counter()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng = sh.engine
eng.set_stream(stream.cuda_stream)
eng.begin()
eng.configure(1 << 40, snp.FirstApplicable())
for _ in range(5):
    eng.launch_step()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(a.steps):
    eng.launch_step()
ev1.record()
torch.cuda.synchronize()
info = eng.info
print(f"world={a.world} rows={a.rows} variant={a.variant}: {ev0.elapsed_time(ev1) / a.steps:.3f} ms/step "
      f"(gen {t1 - t0:.1f} s, build {t2 - t1:.1f} s, tile={info['tile']} n_tiles={info['n_tiles']} "
      f"ring={info['ring_stages']} acc{info['counter_bits']} slots={info['in_edges']})")
