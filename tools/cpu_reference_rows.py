"""The unmodified reference (snpsim 0.1.0 from baseline/_ref) timed on the
GPU box's host cores for the configs beside K3 (BASELINE.md CPU-baseline
plan): K4 (synth 10^7 + delays), K2 (sort n=4096 through the reference's own
gen_sort + prepare, Format.COMPRESSED), K5 (synth 10^8, one step, when host
RAM allows).  Runs on the host only; writes one JSON object.

    python tools/cpu_reference_rows.py [--out profiles/r2_cpu_reference.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402  (reference import + the numpy synth-v1 builder; no repo .so on this path)


def timed(S, prep, steps, workers, sel=None):
    opts = S.SimOptions(max_steps=steps, selection=sel or S.FirstApplicable(), workers=workers)
    t0 = time.perf_counter()
    tr = S.simulate_prepared(prep, opts)
    return time.perf_counter() - t0, tr


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default=None)
    p.add_argument("--k5", action="store_true", help="also K5 (10^8 neurons: ~60 GB of host RAM)")
    a = p.parse_args()
    S = bench.import_reference()
    if S is None:
        print(json.dumps({"unavailable": "reference not installed in baseline/_ref"}))
        return
    host = bench.host_info()
    cores = host["usable_cpus"] or 1
    rows = {"host": host}
    # K4
    t0 = time.perf_counter()
    init, rv, rm, syn = bench.reference_synth(S, 10_000_000, True)
    prep = S.engine.Prepared(bench._Shim(init), S.Format.COMPRESSED, rv, rm, syn)
    gen = time.perf_counter() - t0
    timed(S, prep, 1, cores)
    dt, _ = timed(S, prep, 2, cores)
    dt1, _ = timed(S, prep, 1, 1)
    rows["k4"] = {"s_per_step": dt / 2, "s_per_step_workers1": dt1, "cores": cores, "generate_s": gen,
                  "sample": "synth-v1 q=10^7 + delays 0-3, 2 steps after 1 warm-up (and 1 step with workers=1), "
                            "simulate_prepared via the direct-array shim"}
    del init, rv, rm, syn, prep
    print(json.dumps({"k4": rows["k4"]}), flush=True)
    # K2: the reference's own builder
    t0 = time.perf_counter()
    system = S.gen_sort(S.SortInstance(4096))
    prep = S.prepare(system, S.Format.COMPRESSED)
    build = time.perf_counter() - t0
    dt, tr = timed(S, prep, 20, cores)
    dt1, _ = timed(S, prep, 5, 1)
    rows["k2"] = {"s_per_step": dt / 20, "s_per_step_workers1": dt1 / 5, "cores": cores, "prepare_s": build,
                  "steps_to_halt": 4097, "sample": "sort n=4096 (gen_sort, prepare(Format.COMPRESSED)), the first 20 "
                  "steps with all cores and 5 with workers=1"}
    del system, prep, tr
    print(json.dumps({"k2": rows["k2"]}), flush=True)
    if a.k5:
        t0 = time.perf_counter()
        init, rv, rm, syn = bench.reference_synth(S, 100_000_000, False)
        prep = S.engine.Prepared(bench._Shim(init), S.Format.COMPRESSED, rv, rm, syn)
        gen = time.perf_counter() - t0
        dt, _ = timed(S, prep, 1, cores)
        rows["k5"] = {"s_per_step": dt, "cores": cores, "generate_s": gen,
                      "sample": "synth-v1 q=10^8, one step from the initial configuration (includes the first-step "
                                "page faults), all cores"}
        print(json.dumps({"k5": rows["k5"]}), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(rows, indent=1) + "\n")


if __name__ == "__main__":
    main()
