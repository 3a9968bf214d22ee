"""Measurements for SURVEY 8(f) rows (ingest, trace path, model files):
python tools/measure_next_rows.py > profiles/r1_next_rows.json (on a B200)."""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2408_04343_b200 as snp  # noqa: E402
from paper_2408_04343_b200 import generators as gen  # noqa: E402
from paper_2408_04343_b200 import modelfile as mf  # noqa: E402

out = {}
# CUDA context + module load happen on the first engine; keep them out of the timings
snp.prepare(snp.synth_v1(1000), snp.Format.COMPRESSED)
# ingest: native generator vs numpy restatement, engine creation (device-built layout)
t0 = time.perf_counter(); a = snp.synth_v1(10_000_000); t1 = time.perf_counter()
out["k3_generate_native_s"] = t1 - t0
t0 = time.perf_counter(); gen.synth_v1_numpy(2_000_000); t1 = time.perf_counter()
out["generate_numpy_2e6_s"] = t1 - t0
t0 = time.perf_counter(); prep = snp.prepare(a, snp.Format.COMPRESSED); t1 = time.perf_counter()
out["k3_prepare_s"] = t1 - t0
os.environ["SNPB200_DEVICE_BUILD"] = "0"
t0 = time.perf_counter(); p2 = snp.prepare(a, snp.Format.COMPRESSED); t1 = time.perf_counter()
out["k3_prepare_host_layout_s"] = t1 - t0
del p2
os.environ.pop("SNPB200_DEVICE_BUILD")
# trace path at K3: recorded rows copied vs device digests (20 steps, CONFIGS)
opts = snp.SimOptions(max_steps=20, record=snp.RecordLevel.CONFIGS)
t0 = time.perf_counter(); tr = snp.simulate_prepared(prep, opts); t1 = time.perf_counter()
out["k3_trace_configs_20_steps_s"] = t1 - t0
t0 = time.perf_counter(); dg = snp.trace_digests(prep, opts); t1 = time.perf_counter()
out["k3_trace_digests_20_steps_s"] = t1 - t0
out["digests_match_rows"] = [int(x) for x in dg.configs[:3]] == [snp.row_digest(r) for r in tr.configs[:3]]
with tempfile.TemporaryDirectory() as d:
    path = Path(d) / "t.trace"
    t0 = time.perf_counter(); mf.write_trace(path, tr.configs[:5]); t1 = time.perf_counter()
    out["k3_trace_file_5_rows_native_s"] = t1 - t0
    out["k3_trace_file_5_rows_bytes"] = path.stat().st_size
del tr, prep
# model files at 10^6 neurons (16 M synapses)
m = snp.synth_v1(1_000_000, with_delays=True)
with tempfile.TemporaryDirectory() as d:
    path = Path(d) / "m.snp"
    t0 = time.perf_counter(); mf.save_model(path, m); t1 = time.perf_counter()
    out["model_1e6_save_native_s"] = t1 - t0
    out["model_1e6_bytes"] = path.stat().st_size
    t0 = time.perf_counter(); back = mf.load_model(path); t1 = time.perf_counter()
    out["model_1e6_load_native_s"] = t1 - t0
    out["model_roundtrip_equal"] = bool((back.adj_targets == m.adj_targets).all() and (back.rules.delay == m.rules.delay).all())
print(json.dumps(out, indent=1))
