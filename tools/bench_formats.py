"""Format comparison on the sort family (the paper's Table 4 / Fig. 6 analogue,
PAPER.md:478-506) and small-system step latency, on one B200.

    python tools/bench_formats.py [--sizes 3,10,100,500,2048,4096] [--out profiles/r2_formats.json]

For every sort instance n (worst case n..1, n+1 steps to halt) and every
format/variant that fits the device: engine creation time, device-timed
ms/step over the whole run to halt (CUDA events around the CUDA-graph
replay, snp_time_steps), the step kernel's own per-launch time, SURVEY.md
8(d) algorithmic bytes per step from the kernels' exact counters, and the
device bytes of the engine.  Also a 20-step device-timed segment of K3/K4
for every format.  Numbers printed by this tool are device-timed; none are
taken under a profiler.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2408_04343_b200 as snp  # noqa: E402
from bench import algorithmic_bytes, measured_peaks  # noqa: E402

FORMATS = [("sparse", "auto"), ("ell", "auto"), ("compressed", "tiled"), ("compressed", "pull"),
           ("compressed", "push"), ("compressed", "small")]


def fits(fmt: str, n: int) -> bool:
    m = n * n + 2 * n  # sort family: detectors own n rules each, inputs/outputs one
    q = 3 * n
    if fmt == "sparse":
        return m * q * 4 < 120e9
    if fmt == "ell":
        return m * (n + 2) * 8 < 120e9
    return True


def fits_variant(variant: str, n: int) -> bool:
    return variant != "small" or 3 * n <= 16384


def measure(arrays, fmt: str, variant: str, steps: int, warmup: int = 3) -> dict:
    t0 = time.perf_counter()
    prep = snp.prepare(arrays, snp.Format(fmt), variant=variant)
    prep_s = time.perf_counter() - t0
    eng = prep.engine
    sel = snp.FirstApplicable()
    eng.begin()
    eng.time_steps(min(warmup, steps), sel)
    eng.begin()
    tot, _, res = eng.time_steps(steps, sel)
    eng.begin()
    _, kms, _ = eng.time_steps(steps, sel, per_kernel=True)
    eng.begin()
    _, _, rs = eng.time_steps(steps, sel, collect_stats=True)
    done = int(rs.steps)
    st = rs.stats_dict()
    ns = max(1, int(st.get("steps", steps)))
    alg = algorithmic_bytes(fmt, arrays.neuron_count, arrays.rule_count, st, ns)
    ms = tot / steps
    info = eng.info
    out = {"format": fmt, "variant": variant, "variant_id": int(info["variant"]), "prepare_s": prep_s, "steps": steps,
           "steps_done": done, "ms_per_step": ms, "step_kernel_ms": kms, "launches_per_step": res.kernel_launches / steps,
           "alg_bytes_per_step": alg, "alg_GBps": alg / (ms / 1000) / 1e9,
           "device_MB": info["device_bytes"] / 2**20}
    del prep, eng
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--sizes", default="3,10,100,500,2048,4096")
    p.add_argument("--synth", default="k3,k4")
    p.add_argument("--out", default=None)
    a = p.parse_args()
    hbm = float(measured_peaks()["hbm_gbs"])
    rows = []
    for n in [int(x) for x in a.sizes.split(",") if x]:
        arrays = snp.sort_arrays(snp.SortInstance(n))
        for fmt, var in FORMATS:
            if not fits(fmt, n) or not fits_variant(var, n):
                continue
            r = measure(arrays, fmt, var, n + 1)
            r.update({"workload": f"sort n={n}", "q": arrays.neuron_count, "m": arrays.rule_count,
                      "frac": r["alg_GBps"] / hbm})
            rows.append(r)
            print(json.dumps(r), flush=True)
        del arrays
    for wl in [x for x in a.synth.split(",") if x]:
        arrays = snp.synth_v1(10_000_000, with_delays=wl == "k4")
        for fmt, var in [("ell", "auto"), ("compressed", "tiled"), ("compressed", "pull"), ("compressed", "push")]:
            r = measure(arrays, fmt, var, 20)
            r.update({"workload": wl, "q": arrays.neuron_count, "m": arrays.rule_count, "frac": r["alg_GBps"] / hbm})
            rows.append(r)
            print(json.dumps(r), flush=True)
        del arrays
    if a.out:
        Path(a.out).write_text(json.dumps({"hbm_gbs": hbm, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
