"""Benchmark: SNP steps/s at 10^7 neurons on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload k3|k4|k2|k5] [--format compressed|ell|sparse]
                    [--variant pull|push] [--policy first|seeded] [--extra]

Workload (default, BASELINE.json configs[2], "K3" of SURVEY.md 8): synth-v1,
q = 10^7 neurons, out-degree 16, 4 rules/neuron, no delays, FirstApplicable
selection, Optimized (= COMPRESSED) format.  One bench step = one SNP
transition step (selection + transition + delays + halting test) of the
whole system.  Inputs (the system and its state) are resident in HBM; the
per-step working set (~1.2 GB) is ~10x the 126 MB L2, so no flush is needed.

* value / ms_per_step -- K steps replayed from a CUDA graph, CUDA events on
  the engine stream around the whole segment (max over ranks).
* roofline -- SURVEY.md 8(d) algorithmic bytes per step for the format,
  counted exactly by the kernels' own counters, / mean step-kernel duration
  (per-launch CUDA events), vs MEASURED_PEAKS.json hbm_gbs.
* e2e -- the same metric through the C ABI with HOST buffers: per step one
  snp_run(initial=pinned host config, max_steps=1) -> pinned host config, i.e.
  H2D 8q bytes + one step + D2H 8q bytes.
* cpu_baseline / --impl reference -- the reference's numpy engine restated in
  oracle/snp_oracle.py (VectorEngine, engine.py:192-461) with all host cores
  as its thread-pool workers (engine.py:170-189), timed on a bounded sample.

Multi-GPU (torchrun, N>1): weak scaling -- each rank owns a 10^7-neuron row
shard of an (N x 10^7)-neuron system; the per-step production bits are
exchanged by the step kernels' NVLink peer stores (or, without peer access or
with SNPB200_EXCHANGE=nccl, an NCCL all-gather); paper_2408_04343_b200/
sharded.py.  value is whole-job 10^7-neuron-steps/s.  --workload k5 runs
K5's 10^8-neuron system on one GPU.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

Q_K3 = 10_000_000


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=["k3", "k4", "k2", "k5"], default="k3")
    p.add_argument("--q", type=int, default=Q_K3)
    p.add_argument("--format", choices=["compressed", "ell", "sparse"], default="compressed")
    p.add_argument("--variant", choices=["tiled", "pull", "push"], default="tiled")
    p.add_argument("--policy", choices=["first", "seeded"], default="first")
    p.add_argument("--extra", action="store_true", help="also measure the other formats/policies")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    return p.parse_args()


def measured_peaks() -> dict:
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except FileNotFoundError:
        return {"hbm_gbs": 6650.0, "fallback": True}


def make_workload(args, q=None):
    import paper_2408_04343_b200 as snp
    q = q or args.q
    if args.workload == "k2":
        return snp.sort_arrays(snp.SortInstance(4096)), "sort n=4096 (K2)"
    if args.workload == "k5":
        q = 10 * Q_K3  # K5's 10^8-neuron system on one GPU
    a = snp.synth_v1(q, with_delays=(args.workload == "k4"))
    return a, f"synth-v1 q={q} out-degree 16, 4 rules/neuron{', delays 0-3' if args.workload == 'k4' else ''}"


def selection(args):
    import paper_2408_04343_b200 as snp
    return snp.FirstApplicable() if args.policy == "first" else snp.SeededRandom(240804343)


# -- clocks ------------------------------------------------------------------------------

class ClockSampler:
    """NVML sampling (every 5 ms) of SM clock and clock-event reasons."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int = 0):
        self.samples = []
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception as exc:  # pragma: no cover - no NVML
            self.error = str(exc)
            self.max_mhz = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                try:
                    reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                except AttributeError:
                    reasons = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                self.samples.append((time.perf_counter(), mhz, reasons))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self) -> dict:
        if not self._ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mhz = [s[1] for s in self.samples]
        bits = 0
        for s in self.samples:
            bits |= s[2]
        names = sorted(n for b, n in self.REASONS.items() if bits & b and n != "gpu_idle")
        return {"sm_mhz": float(statistics.median(mhz)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# -- algorithmic bytes --------------------------------------------------------

def algorithmic_bytes(fmt: str, q: int, m: int, st: dict, steps: int) -> float:
    """Per-step compulsory HBM bytes of the format, from the
    kernels' exact counters averaged over ``steps`` steps."""
    scanned = st["scanned"] / steps
    fired = st["fired"] / steps
    rows = st["rows"] / steps
    base = 28.0 * q + 4.0 * scanned
    if fmt == "compressed":
        return base + 12.0 * fired + 4.0 * rows
    if fmt == "ell":
        return base + 4.0 * fired + 8.0 * (fired + rows)
    return base + 4.0 * fired + 4.0 * fired * q  # dense rows actually read (fired rows only)


# -- our arm -----------------------------------------------------------------------------------

def run_ours(args, rank: int, world: int):
    import torch

    import paper_2408_04343_b200 as snp

    torch.cuda.set_device(0 if world == 1 else int(os.environ.get("LOCAL_RANK", rank)))
    sel = selection(args)
    t0 = time.perf_counter()
    arrays, desc = make_workload(args)
    gen_s = time.perf_counter() - t0
    fmt = snp.Format(args.format)
    t0 = time.perf_counter()
    prep = snp.prepare(arrays, fmt, variant=args.variant if fmt is snp.Format.COMPRESSED else "auto",
                       device=torch.cuda.current_device())
    prep_s = time.perf_counter() - t0
    eng = prep.engine
    q, m = arrays.neuron_count, arrays.rule_count

    # warm-up W steps, then exactly K timed steps (CUDA events on the engine stream)
    eng.begin()
    eng.time_steps(args.warmup, sel)
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        total_ms, _, res = eng.time_steps(args.steps, sel)
    torch.cuda.synchronize()
    launches = int(res.kernel_launches)

    # per-launch durations of the step kernel (CUDA events around each launch)
    eng.begin()
    eng.time_steps(args.warmup, sel)
    nk = min(args.steps, 50)
    _, kernel_ms, _ = eng.time_steps(nk, sel, per_kernel=True)
    # exact traffic counters of the same steps (separate pass: counting costs atomics)
    eng.begin()
    eng.time_steps(args.warmup, sel)
    _, _, res_k = eng.time_steps(nk, sel, collect_stats=True)
    stats = res_k.stats_dict()
    alg = algorithmic_bytes(args.format, q, m, stats, nk)

    # e2e through the C ABI with pinned host buffers: one step per call
    host_in = torch.from_numpy(arrays.initial.copy()).pin_memory()
    host_out = torch.empty(q, dtype=torch.int64).pin_memory()
    import ctypes

    from paper_2408_04343_b200 import _native as nat
    opts = eng._opts(1, sel)
    r = nat.Result()
    lib = nat.load()
    e2e_steps = max(3, min(args.steps, 30))
    for _ in range(2):
        lib.snp_run(eng._h, ctypes.c_void_p(host_in.data_ptr()), ctypes.byref(opts),
                    ctypes.c_void_p(host_out.data_ptr()), None, ctypes.byref(r))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        rc = lib.snp_run(eng._h, ctypes.c_void_p(host_in.data_ptr()), ctypes.byref(opts),
                         ctypes.c_void_p(host_out.data_ptr()), None, ctypes.byref(r))
        nat.check(rc)
        host_in, host_out = host_out, host_in  # the result feeds the next step
    e2e_s = time.perf_counter() - t0
    # the same C-ABI call as one simulation of K steps (host config in, host
    # final config out), which is how simulate_prepared is used
    opts_k = eng._opts(args.steps, sel)
    t0 = time.perf_counter()
    nat.check(lib.snp_run(eng._h, ctypes.c_void_p(host_in.data_ptr()), ctypes.byref(opts_k),
                          ctypes.c_void_p(host_out.data_ptr()), None, ctypes.byref(r)))
    e2e_run_s = time.perf_counter() - t0

    return {
        "q": q, "m": m, "desc": desc, "gen_s": gen_s, "prep_s": prep_s, "total_ms": total_ms,
        "kernel_ms": kernel_ms, "stats": stats, "stats_steps": nk, "alg_bytes": alg,
        "clocks": clk.summary(), "launches": launches, "info": eng.info,
        "e2e_steps_per_s": e2e_steps / e2e_s, "e2e_bytes": 8 * q, "arrays": arrays,
        "e2e_run_steps_per_s": args.steps / e2e_run_s,
    }


# -- CPU leg -----------------------------------------------------------------------------------

def cpu_port(args, steps: int, q: int | None = None):
    """The reference's vectorised engine (oracle/snp_oracle.py VectorEngine)."""
    from oracle.snp_oracle import OracleSystem, VectorEngine
    arrays, _ = make_workload(args, q)
    s = OracleSystem.from_arrays(arrays)
    cores = os.cpu_count() or 1
    pol, seed = (0, 0) if args.policy == "first" else (1, 240804343)
    ve = VectorEngine(s, args.format, workers=cores)
    cfg = s.initial.copy()
    dly = np.zeros(s.q, dtype=np.int64)

    def one_step(k, cfg, dly):
        ch = ve.sv_calc(cfg, dly, pol, seed, k)
        nxt = ve.step(cfg, dly, ch)
        return nxt, ve.update_delays(dly, ch)

    cfg, dly = one_step(0, cfg, dly)  # warm-up (page faults, pool start)
    t0 = time.perf_counter()
    for k in range(1, steps + 1):
        cfg, dly = one_step(k, cfg, dly)
    dt = (time.perf_counter() - t0) / steps
    return dt, cores, s.q


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if (args.gpus > 1 or world > 1) and args.impl == "ours":
        from paper_2408_04343_b200.sharded import bench_sharded
        return bench_sharded(args, rank, world)

    metric = "SNP steps/sec at 10^7 neurons"
    unit = "steps/s"
    if args.workload == "k2":
        metric, unit = "SNP steps/sec, sort n=4096", "steps/s"
    if args.workload == "k5":
        metric, unit = "SNP steps/sec at 10^8 neurons (one GPU)", "steps/s"
    config = {"workload": "", "format": args.format, "variant": args.variant, "policy": args.policy,
              "l2": "working set >> 126 MB L2 (no flush needed)", "parallelism": f"rows/{args.gpus}"}

    if args.impl == "reference":
        if rank != 0:
            return  # the CPU reference runs once, on rank 0
        args.q = Q_K3  # the metric is quoted per 10^7 neurons whatever N is
        # bounded sample: whole run within a few minutes
        n = args.steps + args.warmup
        q_s = args.q if n <= 6 else max(1_000_000, int(args.q * 6 / n) // 1000 * 1000)
        dt, cores, qs = cpu_port(args, max(1, args.steps), q_s)
        scale = qs / args.q
        v = scale / dt
        config["workload"] = f"synth-v1 q={args.q} (K3), sampled at q={qs}"
        line = {
            "impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic", "config": config,
            "cpu_baseline": {"value": v, "unit": unit, "cores": cores, "kind": "port",
                             "sample": f"{args.steps} steps of a q={qs} synth-v1 system, scaled by {scale:g} to q={args.q}"},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return

    r = run_ours(args, rank, world)
    peaks = measured_peaks()
    hbm = float(peaks["hbm_gbs"])
    value = args.steps / (r["total_ms"] / 1000.0)
    achieved = r["alg_bytes"] / (r["kernel_ms"] / 1000.0) / 1e9
    config["workload"] = r["desc"]
    config["q"] = r["q"]
    config["m"] = r["m"]
    line = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["total_ms"] / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic (synth-v1, counter-based)",
        "config": config,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": None, "peak_source": "measured" if "fallback" not in peaks else "fallback",
                     "alg_bytes_per_step": r["alg_bytes"], "kernel_ms": r["kernel_ms"],
                     "frac_of_8TBps_nominal": achieved / 8000.0},
        "e2e": {"value": r["e2e_steps_per_s"], "unit": unit, "h2d_bytes_per_step": r["e2e_bytes"],
                "d2h_bytes_per_step": r["e2e_bytes"], "path": "snp_run C ABI, pinned host buffers, 1 step/call",
                "run_value": r["e2e_run_steps_per_s"],
                "run_path": f"one snp_run call of {args.steps} steps, host config in / final config out"},
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "counters_per_step": {k: v / r["stats_steps"] for k, v in r["stats"].items() if k != "steps"},
        "setup_s": {"generate": r["gen_s"], "prepare": r["prep_s"]},
        "device_bytes": r["info"]["device_bytes"],
    }
    traffic = ROOT / "profiles" / "traffic_bytes.json"
    if traffic.exists():
        try:
            t = json.loads(traffic.read_text())
            line["roofline"]["traffic"] = t.get(f"{args.workload}/{args.format}/{args.variant}/{args.policy}")
        except ValueError:
            pass
    if args.extra:
        line["extra"] = extra_measurements(args)
    if not args.no_cpu:
        n_cpu = 2
        dt, cores, qs = cpu_port(args, n_cpu)
        line["cpu_baseline"] = {"value": (qs / args.q) / dt, "unit": unit, "cores": cores, "kind": "port",
                                "sample": f"{n_cpu} steps (after 1 warm-up) of the same q={qs} system, "
                                          f"numpy VectorEngine with {cores} thread-pool workers"}
    print(json.dumps(line))


def extra_measurements(args) -> dict:
    """Other formats / policies / K4 on the same box (not the headline)."""
    import paper_2408_04343_b200 as snp
    out = {}
    cases = [("k3", "compressed", "pull", "first"), ("k3", "compressed", "push", "first"),
             ("k3", "ell", "push", "first"), ("k3", "compressed", "tiled", "seeded"),
             ("k4", "compressed", "tiled", "first"), ("k4", "compressed", "tiled", "seeded"),
             ("k2", "compressed", "tiled", "first"), ("k2", "compressed", "pull", "first"),
             ("k5", "compressed", "tiled", "first")]
    for wl, fmt, var, pol in cases:
        a2 = argparse.Namespace(**vars(args))
        a2.workload, a2.format, a2.variant, a2.policy = wl, fmt, var, pol
        arrays, _ = make_workload(a2)
        prep = snp.prepare(arrays, snp.Format(fmt), variant=var if fmt == "compressed" else "auto")
        sel = selection(a2)
        eng = prep.engine
        eng.begin()
        eng.time_steps(args.warmup, sel)
        tot, _, _ = eng.time_steps(args.steps, sel)
        eng.begin()
        eng.time_steps(args.warmup, sel)
        _, kms, _ = eng.time_steps(30, sel, per_kernel=True)
        eng.begin()
        eng.time_steps(args.warmup, sel)
        _, _, res = eng.time_steps(30, sel, collect_stats=True)
        alg = algorithmic_bytes(fmt, arrays.neuron_count, arrays.rule_count, res.stats_dict(), 30)
        ms = tot / args.steps
        out[f"{wl}/{fmt}/{var}/{pol}"] = {"steps_per_s": 1000.0 / ms, "ms_per_step": ms, "step_kernel_ms": kms,
                                          "alg_bytes_per_step": alg, "alg_GBps_per_step": alg / (ms / 1000) / 1e9,
                                          "neurons": arrays.neuron_count}
        del prep, eng, arrays
    return out


if __name__ == "__main__":
    main()
