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
* cpu_baseline / --impl reference -- the reference itself (snpsim 0.1.0,
  unmodified, installed into baseline/_ref) on the same full-size workload:
  its simulate_prepared (engine.py:416-461) over the direct-array Prepared
  shim, all host cores as its thread-pool workers (engine.py:170-189).
  --impl reference times W + K full-size steps (fewer timed steps only if K
  would not fit the time budget; never a smaller system); cpu_baseline is a
  2-step sample plus one workers=1 step.

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
    # the same one-step calls with device buffers (torch CUDA tensors through
    # unified addressing: device-to-device copies instead of PCIe)
    dev_in = torch.from_numpy(arrays.initial.copy()).cuda()
    dev_out = torch.empty(q, dtype=torch.int64, device="cuda")
    for _ in range(2):
        nat.check(lib.snp_run(eng._h, ctypes.c_void_p(dev_in.data_ptr()), ctypes.byref(opts),
                              ctypes.c_void_p(dev_out.data_ptr()), None, ctypes.byref(r)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        nat.check(lib.snp_run(eng._h, ctypes.c_void_p(dev_in.data_ptr()), ctypes.byref(opts),
                              ctypes.c_void_p(dev_out.data_ptr()), None, ctypes.byref(r)))
        dev_in, dev_out = dev_out, dev_in
    e2e_dev_s = time.perf_counter() - t0

    return {
        "q": q, "m": m, "desc": desc, "gen_s": gen_s, "prep_s": prep_s, "total_ms": total_ms,
        "kernel_ms": kernel_ms, "stats": stats, "stats_steps": nk, "alg_bytes": alg,
        "clocks": clk.summary(), "launches": launches, "info": eng.info,
        "e2e_steps_per_s": e2e_steps / e2e_s, "e2e_bytes": 8 * q, "arrays": arrays,
        "e2e_run_steps_per_s": args.steps / e2e_run_s, "e2e_device_steps_per_s": e2e_steps / e2e_dev_s,
    }


# -- CPU leg: the unmodified reference (baseline/_ref) ------------------------------------

REF_DIR = ROOT / "baseline" / "_ref"


_REF_MOD = None


def import_reference():
    """The reference package ``snpsim`` as installed (unmodified) into
    baseline/_ref, or None.  Nothing of this repo is imported on that path.
    Loaded under its own name even when ``snpsim`` is already aliased in
    this process (the conformance tests alias it to the drop-in); callers
    reach its submodules as attributes (``snpsim.engine``, ...)."""
    global _REF_MOD
    if _REF_MOD is not None:
        return _REF_MOD
    if not (REF_DIR / "snpsim").is_dir():
        return None
    ours = lambda k: k == "snpsim" or k.startswith("snpsim.")  # noqa: E731
    saved = {k: sys.modules.pop(k) for k in list(sys.modules) if ours(k)}
    sys.path.insert(0, str(REF_DIR))
    try:
        import snpsim
        loaded = [k for k in sys.modules if ours(k)]
    finally:
        sys.path.remove(str(REF_DIR))
    if saved:  # put the alias back; the reference stays reachable through _REF_MOD
        for k in loaded:
            sys.modules.pop(k, None)
        sys.modules.update(saved)
    _REF_MOD = snpsim
    return snpsim


class _Shim:
    """The only system fields the reference's simulate_prepared reads
    (engine.py:427-428): the direct-array method of SURVEY.md 8(c)."""

    def __init__(self, initial):
        self.initial_spikes = initial
        self.neuron_count = len(initial)


def reference_synth(snpsim, q: int, with_delays: bool, seed: int = 240804343):
    """synth-v1 built with numpy and the reference's own
    mix64_array (selection.py:48-62) straight into the reference's
    RuleVector / NeuronRuleMap / SynapseMatrix (matrices.py:48-112); the same
    system as paper_2408_04343_b200.synth_v1 (tests/test_oracle_golden.py)."""
    NeuronRuleMap, RuleVector = snpsim.matrices.NeuronRuleMap, snpsim.matrices.RuleVector
    SynapseMatrix, mix64_array = snpsim.matrices.SynapseMatrix, snpsim.selection.mix64_array
    idx = np.arange(q, dtype=np.int64)
    h = lambda stream: mix64_array(seed, stream, idx)  # noqa: E731
    init = (h(0) % np.uint64(8)).astype(np.int64)
    deg, width = 16, (q - 1) // 16
    tg = np.empty((deg, q), dtype=np.int64)
    for k in range(deg):
        tg[k] = (idx + 1 + k * width + (h(1 + k) % np.uint64(width)).astype(np.int64)) % q
    tg.sort(axis=0)
    t0 = 2 + (h(17) % np.uint64(4)).astype(np.int64)
    t1 = 3 + (h(18) % np.uint64(6)).astype(np.int64)
    c1 = 1 + (h(19) % t1.astype(np.uint64)).astype(np.int64)
    t2 = 1 + (h(20) % np.uint64(5)).astype(np.int64)
    one = np.ones(q, np.int64)
    thr = np.stack([t0, t1, t2, one], axis=1).reshape(-1)
    cons = np.stack([t0, c1, t2, one], axis=1).reshape(-1)
    prod = np.tile(np.array([1, 1, 0, 1], np.int64), q)
    exact = np.tile(np.array([True, False, True, False]), q)
    dly = np.zeros((q, 4), np.int64)
    if with_delays:
        for r, stream in ((0, 21), (1, 22), (3, 23)):
            dly[:, r] = (h(stream) % np.uint64(4)).astype(np.int64)
    rv = RuleVector(thr, exact, cons, prod, dly.reshape(-1), np.repeat(idx, 4))
    rm = NeuronRuleMap(np.arange(0, 4 * q + 1, 4, dtype=np.int64))
    return init, rv, rm, SynapseMatrix(tg)


def host_info() -> dict:
    model, mem_gb = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem_gb = round(int(line.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "usable_cpus": usable, "ram_gb": mem_gb,
            "numpy": np.__version__, "python": sys.version.split()[0]}


class ReferenceArm:
    """The reference's own engine (snpsim.engine.simulate_prepared,
    engine.py:416-461, unmodified, from baseline/_ref) on the bench workload,
    driven through the direct-array Prepared shim.  One simulate_prepared
    call of K steps from the initial configuration is one timed run, exactly
    how the reference's own harness times it (bench.py:80-96)."""

    def __init__(self, args):
        self.snpsim = import_reference()
        if self.snpsim is None:
            raise RuntimeError(f"reference not installed at {REF_DIR}")
        S = self.snpsim
        ref_engine = S.engine
        q = Q_K3 if args.workload in ("k3", "k4") else args.q
        t0 = time.perf_counter()
        init, rv, rm, syn = reference_synth(S, q, args.workload == "k4")
        self.gen_s = time.perf_counter() - t0
        self.q = q
        self.prep = ref_engine.Prepared(_Shim(init), S.Format.COMPRESSED, rv, rm, syn)
        self.sel = S.FirstApplicable() if args.policy == "first" else S.SeededRandom(240804343)

    def run(self, steps: int, workers: int) -> float:
        """Wall seconds of one simulate_prepared run of ``steps`` steps."""
        S = self.snpsim
        opts = S.SimOptions(max_steps=steps, selection=self.sel, workers=workers)
        t0 = time.perf_counter()
        tr = S.simulate_prepared(self.prep, opts)
        dt = time.perf_counter() - t0
        assert tr.steps == steps, (tr.steps, steps)
        return dt


def cpu_reference_sample(args, steps: int = 2) -> dict:
    """cpu_baseline of the GPU arm: the unmodified reference on the same
    full-size workload, all host cores (plus one workers=1 step), a bounded
    sample of ~10-30 s of CPU work."""
    if args.workload not in ("k3", "k4") or import_reference() is None:
        return cpu_port_sample(args, steps)
    arm = ReferenceArm(args)
    cores = host_info()["usable_cpus"] or 1
    arm.run(1, cores)  # warm-up: page faults, thread pool
    dt = arm.run(steps, cores) / steps
    dt1 = arm.run(1, 1)
    return {"value": 1.0 / dt, "unit": "steps/s", "cores": cores, "kind": "reference",
            "sample": f"{steps} full steps of the same q={arm.q} system through the unmodified reference "
                      f"(baseline/_ref snpsim {getattr(arm.snpsim, '__version__', '0.1.0')} simulate_prepared, "
                      f"direct-array shim, workers={cores}) after 1 warm-up step",
            "workers1_value": 1.0 / dt1, "host": host_info()}


def cpu_port_sample(args, steps: int = 2) -> dict:
    """Fallback when the reference is not installed: the numpy restatement
    (oracle/snp_oracle.py VectorEngine) of the same engine."""
    from oracle.snp_oracle import OracleSystem, VectorEngine
    arrays, _ = make_workload(args)
    s = OracleSystem.from_arrays(arrays)
    cores = host_info()["usable_cpus"] or 1
    pol, seed = (0, 0) if args.policy == "first" else (1, 240804343)
    ve = VectorEngine(s, args.format, workers=cores)
    cfg = s.initial.copy()
    dly = np.zeros(s.q, dtype=np.int64)

    def one_step(k, cfg, dly):
        ch = ve.sv_calc(cfg, dly, pol, seed, k)
        return ve.step(cfg, dly, ch), ve.update_delays(dly, ch)

    cfg, dly = one_step(0, cfg, dly)
    t0 = time.perf_counter()
    for k in range(1, steps + 1):
        cfg, dly = one_step(k, cfg, dly)
    dt = (time.perf_counter() - t0) / steps
    return {"value": 1.0 / dt, "unit": "steps/s", "cores": cores, "kind": "port",
            "sample": f"{steps} steps of the same q={s.q} system, numpy VectorEngine ({cores} workers)",
            "host": host_info()}


def reference_main(args, metric: str, unit: str, config: dict) -> None:
    """bench.py --impl reference: W warm-up steps, then K timed full-size
    steps of the unmodified reference on this box's host cores (one
    simulate_prepared run each).  If K steps would not finish within the
    time budget, fewer full-size steps are timed (``steps_timed``); nothing
    is sampled at a smaller size or extrapolated."""
    budget_s = float(os.environ.get("SNPB200_REF_BUDGET_S", "240"))
    cores = host_info()["usable_cpus"] or 1
    if args.workload not in ("k3", "k4") or import_reference() is None:
        why = "reference not installed in baseline/_ref" if import_reference() is None else \
            f"--impl reference is defined for the K3/K4 workloads (got {args.workload})"
        print(json.dumps({"impl": "reference", "unavailable": why}))
        return
    t0 = time.perf_counter()
    arm = ReferenceArm(args)
    setup_s = time.perf_counter() - t0
    w = max(1, args.warmup)
    t_w = arm.run(w, cores)
    per = t_w / w
    k = args.steps
    left = budget_s - (time.perf_counter() - t0)
    if k * per > left:
        k = max(1, int(left / per))
    dt = arm.run(k, cores)
    v = k / dt
    config["workload"] = f"synth-v1 q={arm.q} out-degree 16, 4 rules/neuron" + \
        (", delays 0-3" if args.workload == "k4" else "")
    config["q"] = arm.q
    config["m"] = 4 * arm.q
    line = {
        "impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": args.gpus,
        "steps": args.steps, "steps_timed": k, "warmup": w, "ms_per_step": 1000.0 * dt / k,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (synth-v1 via numpy + the reference's mix64_array)", "config": config,
        "cpu_baseline": {"value": v, "unit": unit, "cores": cores, "kind": "reference",
                         "sample": f"{k} full-size steps in one simulate_prepared run (after a {w}-step run), "
                                   f"unmodified snpsim from baseline/_ref, workers={cores}",
                         "host": host_info()},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": {"generate_and_shim": setup_s, "generate": arm.gen_s},
        "path": "snpsim.simulate_prepared (engine.py:416-461) via Prepared(_Shim, COMPRESSED, RuleVector, "
                "NeuronRuleMap, SynapseMatrix)",
    }
    print(json.dumps(line))


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
        return reference_main(args, metric, unit, config)

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
                "run_path": f"one snp_run call of {args.steps} steps, host config in / final config out",
                "device_value": r["e2e_device_steps_per_s"],
                "device_path": "the same 1-step snp_run calls with CUDA-tensor buffers (device-to-device copies)"},
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
        line["cpu_baseline"] = cpu_reference_sample(args)
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
