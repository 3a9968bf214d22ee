"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): python tools/sanitize_smoke.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2408_04343_b200 as snp  # noqa: E402
from paper_2408_04343_b200 import sharded as shd  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from conftest import concentrated_system, multi_amount_system  # noqa: E402

a = snp.synth_v1(3000, with_delays=True)
sort = snp.sort_arrays(snp.SortInstance(40))
for arrays in (a, sort):
    for fmt, var in [(snp.Format.COMPRESSED, "tiled"), (snp.Format.COMPRESSED, "tiled2"),
                     (snp.Format.COMPRESSED, "pull"), (snp.Format.COMPRESSED, "push"),
                     (snp.Format.COMPRESSED, "small"),
                     (snp.Format.ELL, "auto"), (snp.Format.SPARSE, "auto")]:
        prep = snp.prepare(arrays, fmt, variant=var)
        for sel in (snp.FirstApplicable(), snp.SeededRandom(3)):
            snp.run_final(prep, snp.SimOptions(max_steps=6, selection=sel))
            snp.simulate_prepared(prep, snp.SimOptions(max_steps=4, selection=sel, record=snp.RecordLevel.FULL))
        print("ok", arrays.neuron_count, fmt.value, var, flush=True)
    snp.trace_digests(snp.prepare(arrays, snp.Format.COMPRESSED),
                      snp.SimOptions(max_steps=4, record=snp.RecordLevel.FULL))
# binned push: every delivery into one tile (bucket overflow), and u32 entries (mixed amounts)
for arrays in (concentrated_system(5000), multi_amount_system(3000, 300)):
    for fmt, var in [(snp.Format.ELL, "auto"), (snp.Format.COMPRESSED, "push")]:
        prep = snp.prepare(arrays, fmt, variant=var)
        snp.run_final(prep, snp.SimOptions(max_steps=6, selection=snp.SeededRandom(3)))
        print("ok binned", arrays.neuron_count, fmt.value, var, prep.engine.info["push_kernel"], flush=True)
# row partition, peer exchange in one process
import torch  # noqa: E402
q = a.neuron_count
L = shd.shard_layout(q, 2)
ranks = [shd.ShardedEngine(shd.local_arrays(a, L, r), q, r, 2) for r in range(2)]
shd.ShardedEngine.connect_local(ranks)
st = torch.cuda.Stream()
for r in ranks:
    r.engine.set_stream(st.cuda_stream)
    r.engine.begin()
    r.engine.configure(5, snp.FirstApplicable())
for _ in range(6):
    for r in ranks:
        r.engine.launch_step()
torch.cuda.synchronize()
print("ok sharded p2p", [int(r.engine.poll().halt) for r in ranks])
