"""Simulation engine -- drop-in for ``snpsim.engine`` running on B200.

Reference: ``pkg/src/snpsim/engine.py``.  Same public names, argument meaning,
trace semantics and exceptions:

* ``prepare`` (engine.py:388-402)  -> builds the device engine through the C
  ABI (``snp_engine_create``); the reference's host matrices are *not*
  materialised (``Prepared.matrix`` builds them lazily on request).
* ``simulate`` / ``simulate_prepared`` (:405-461) -> ``snp_begin`` +
  ``snp_advance`` segments; the whole loop (selection, transition, delays,
  halting) runs on the device; rows of the trace are copied out per segment.
* ``sv_calc`` (:192-236), ``step_sparse`` / ``step_ell`` / ``step_compressed``
  (:239-355), ``update_delays`` (:358-366) -> ``snp_sv_calc`` / ``snp_step``
  / ``snp_update_delays`` (same kernels as the run loop).
* ``NegativeSpikes`` (:48-54) is raised from the device error word; the run
  is aborted with no partial trace, as in the reference.

``SimOptions.workers`` is accepted and validated (>= 1) for compatibility;
the GPU grid replaces the reference's thread-pool chunking, and results do
not depend on it (as in the reference, engine.py:15-17).

Differences (documented in INTEGRATION.md): ``Format.ORACLE`` is the
reference's CPU interpreter; it is test infrastructure here (``oracle/``),
so ``prepare(..., Format.ORACLE)`` raises ``ValueError``.  Extensions:
``variant`` on ``prepare`` (COMPRESSED: "tiled" (default), "pull", or the
paper's "push"), and
``run_final`` (final state + traffic counters, no per-step trace).
"""

from __future__ import annotations

import enum
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .generators import SystemArrays, system_arrays
from .matrices import (
    EllMatrix,
    Format,
    NeuronRuleMap,
    RuleVector,
    SparseMatrix,
    SynapseMatrix,
    compressed_from_arrays,
    ell_from_arrays,
    offsets_from_owners,
    sparse_from_arrays,
)
from .model import SNPSystem
from .selection import FirstApplicable, Selection, policy_code


class EngineError(Exception):
    """Base class for simulation-time failures."""


class NegativeSpikes(EngineError):
    """A step drove some neuron's spike count below zero (engine.py:48-54)."""


class HaltReason(enum.Enum):
    STEP_LIMIT = "step_limit"
    NO_APPLICABLE_RULES = "no_applicable_rules"


class RecordLevel(enum.Enum):
    CONFIGS = "configs"
    CONFIGS_AND_DELAYS = "configs+delays"
    FULL = "full"


_REC_FLAGS = {
    RecordLevel.CONFIGS: nat.SNP_REC_CONFIGS,
    RecordLevel.CONFIGS_AND_DELAYS: nat.SNP_REC_CONFIGS | nat.SNP_REC_DELAYS,
    RecordLevel.FULL: nat.SNP_REC_CONFIGS | nat.SNP_REC_DELAYS | nat.SNP_REC_SPIKING,
}
_FMT_CODES = {Format.SPARSE: nat.SNP_FMT_SPARSE, Format.ELL: nat.SNP_FMT_ELL,
              Format.COMPRESSED: nat.SNP_FMT_COMPRESSED}
_VARIANTS = {"auto": nat.SNP_VARIANT_AUTO, "pull": nat.SNP_VARIANT_PULL, "push": nat.SNP_VARIANT_PUSH,
             "tiled": nat.SNP_VARIANT_TILED, "tiled2": nat.SNP_VARIANT_TILED2, "small": nat.SNP_VARIANT_SMALL}


@dataclass(frozen=True)
class SpikingVector:
    """``chosen[i]``: global rule id neuron ``i`` fires, or -1."""

    chosen: np.ndarray  # int64[q]

    def flags(self, rule_count: int) -> np.ndarray:
        out = np.zeros(rule_count, dtype=np.uint8)
        out[self.chosen[self.chosen >= 0]] = 1
        return out

    @property
    def is_empty(self) -> bool:
        return bool((self.chosen < 0).all())

    def fired_rules(self) -> np.ndarray:
        return np.sort(self.chosen[self.chosen >= 0])


@dataclass
class SimState:
    config: np.ndarray
    delays: np.ndarray
    spiking: SpikingVector | None = None
    step: int = 0


@dataclass(frozen=True)
class SimOptions:
    max_steps: int
    selection: Selection = field(default_factory=FirstApplicable)
    record: RecordLevel = RecordLevel.CONFIGS
    workers: int = 1

    def __post_init__(self):
        if self.max_steps < 1:
            raise ValueError(f"max_steps must be >= 1, got {self.max_steps}")
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")


@dataclass(eq=False)
class Trace:
    """``configs[k]`` = configuration after ``k`` steps (engine.py:129-159)."""

    configs: list[np.ndarray]
    halt_reason: HaltReason
    delays: list[np.ndarray] | None = None
    spiking: list[np.ndarray] | None = None

    @property
    def steps(self) -> int:
        return len(self.configs) - 1

    def __eq__(self, other) -> bool:
        if not isinstance(other, Trace):
            return NotImplemented
        if self.halt_reason is not other.halt_reason:
            return False
        pairs = [(self.configs, other.configs), (self.delays, other.delays),
                 (self.spiking, other.spiking)]
        for mine, theirs in pairs:
            if (mine is None) != (theirs is None):
                return False
            if mine is not None and not _same_rows(mine, theirs):
                return False
        return True


def _same_rows(a, b) -> bool:
    return len(a) == len(b) and all(np.array_equal(x, y) for x, y in zip(a, b))


def format_trace(trace: Trace) -> str:
    """One configuration per line, space-separated (engine.py:162-165)."""
    return "".join(" ".join(map(str, np.asarray(c).tolist())) + "\n" for c in trace.configs)


# -- device engine --------------------------------------------------------------

def _c64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


class DeviceEngine:
    """Owner of one ``snp_engine`` handle (device layouts + run state)."""

    def __init__(self, fmt: Format, q: int, rules: RuleVector, offsets: np.ndarray,
                 initial: np.ndarray | None = None, *, adj: tuple[np.ndarray, np.ndarray] | None = None,
                 syn: SynapseMatrix | None = None, ell: EllMatrix | None = None,
                 sparse: SparseMatrix | None = None, variant: str = "auto", device: int = 0,
                 world: int = 1, rank: int = 0, x_pbits: int = 0, x_pmax: int = 0):
        if fmt not in _FMT_CODES:
            raise ValueError(f"no device backend for format {fmt!r}")
        if variant not in _VARIANTS:
            raise ValueError(f"variant must be one of {sorted(_VARIANTS)}, got {variant!r}")
        lib = nat.load()
        self.fmt = fmt
        self.q = int(q)
        self.m = len(rules)
        # keep every array alive for the duration of the create call
        keep = {
            "initial": _c64(initial if initial is not None else np.zeros(self.q, dtype=np.int64)),
            "offsets": _c64(offsets), "threshold": _c64(rules.threshold),
            "is_exact": np.ascontiguousarray(rules.is_exact, dtype=np.uint8),
            "consumed": _c64(rules.consumed), "produced": _c64(rules.produced), "delay": _c64(rules.delay),
        }
        d = nat.SystemDesc()
        d.format = _FMT_CODES[fmt]
        d.variant = _VARIANTS[variant]
        d.q, d.m = self.q, self.m
        d.initial = nat.i64p(keep["initial"])
        d.offsets = nat.i64p(keep["offsets"])
        d.threshold = nat.i64p(keep["threshold"])
        d.is_exact = nat.u8p(keep["is_exact"])
        d.consumed = nat.i64p(keep["consumed"])
        d.produced = nat.i64p(keep["produced"])
        d.delay = nat.i64p(keep["delay"])
        if adj is not None:
            keep["adj_off"], keep["adj_dst"] = _c64(adj[0]), _c64(adj[1])
            d.adj_offsets, d.adj_targets = nat.i64p(keep["adj_off"]), nat.i64p(keep["adj_dst"])
        if syn is not None:
            keep["syn"] = _c64(syn.target)
            d.syn_target, d.syn_rows = nat.i64p(keep["syn"]), syn.rows
        if ell is not None:
            keep["ell_t"], keep["ell_a"] = _c64(ell.target), _c64(ell.amount)
            d.ell_target, d.ell_amount, d.ell_rows = nat.i64p(keep["ell_t"]), nat.i64p(keep["ell_a"]), ell.rows
        if sparse is not None:
            keep["sparse"] = _c64(sparse.data)
            d.sparse_data = nat.i64p(keep["sparse"])
        d.device = device
        d.world, d.rank = int(world), int(rank)
        d.x_pbits, d.x_pmax = int(x_pbits), int(x_pmax)
        handle = nat.ctypes.c_void_p()
        rc = lib.snp_engine_create(nat.ctypes.byref(d), nat.ctypes.byref(handle))
        if rc == nat.SNP_ERR_BAD_ARG:
            raise ValueError(lib.snp_last_error().decode())
        if rc == nat.SNP_ERR_CAPACITY:
            raise MemoryError(lib.snp_last_error().decode())
        nat.check(rc)
        self._lib = lib
        self._h = handle
        info = nat.EngineInfo()
        nat.check(lib.snp_engine_get_info(self._h, nat.ctypes.byref(info)))
        self.info = {name: getattr(info, name) for name, _ in nat.EngineInfo._fields_}
        self.q = int(info.q)  # a row-partitioned engine holds only its own rows

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.snp_engine_destroy(h)
            self._h = None

    # -- run loop -------------------------------------------------------------

    def _opts(self, max_steps: int, selection: Selection, record: int = 0, chunk: int = 0,
              use_graph: bool = True, collect_stats: bool = False) -> nat.RunOpts:
        policy, seed = policy_code(selection)
        o = nat.RunOpts()
        o.max_steps, o.policy, o.record, o.seed = int(max_steps), policy, record, seed
        o.chunk, o.use_graph, o.collect_stats = int(chunk), int(bool(use_graph)), int(bool(collect_stats))
        return o

    def _raise(self, rc: int, res: nat.Result | None = None):
        msg = self._lib.snp_last_error().decode()
        if rc == nat.SNP_ERR_NEGATIVE:
            raise NegativeSpikes(msg)
        if rc == nat.SNP_ERR_BAD_ARG:
            raise ValueError(msg)
        if rc == nat.SNP_ERR_CAPACITY:
            raise MemoryError(msg)
        raise nat.NativeError(rc, msg)

    def begin(self, initial: np.ndarray | None = None) -> None:
        arr = None if initial is None else _c64(initial)
        rc = self._lib.snp_begin(self._h, nat.ptr(arr))
        if rc:
            self._raise(rc)

    def trace(self, options: SimOptions, initial: np.ndarray | None = None,
              rows_per_call: int | None = None) -> Trace:
        """The reference's ``simulate_prepared`` loop, recorded."""
        q = self.q
        flags = _REC_FLAGS[options.record]
        self.begin(initial)
        total_rows = options.max_steps + 1
        if rows_per_call is None:
            rows_per_call = int(max(1, min(total_rows, (256 << 20) // max(1, 24 * q))))
        opts = self._opts(options.max_steps, options.selection, record=flags)
        configs, delays, spiking = [], [], []
        want_d = bool(flags & nat.SNP_REC_DELAYS)
        want_s = bool(flags & nat.SNP_REC_SPIKING)
        res = nat.Result()
        while True:
            cap = rows_per_call
            cbuf = np.empty((cap, q), dtype=np.int64)
            dbuf = np.empty((cap, q), dtype=np.int64) if want_d else None
            sbuf = np.empty((cap, q), dtype=np.int64) if want_s else None
            tr = nat.TraceOut()
            tr.configs, tr.delays, tr.spiking = nat.i64p(cbuf), nat.i64p(dbuf), nat.i64p(sbuf)
            tr.cap = cap
            rc = self._lib.snp_advance(self._h, nat.ctypes.byref(opts), cap, nat.ctypes.byref(tr),
                                       nat.ctypes.byref(res))
            if rc:
                self._raise(rc, res)
            configs.extend(cbuf[: tr.config_rows])
            if want_d:
                delays.extend(dbuf[: tr.config_rows])
            if want_s:
                spiking.extend(sbuf[: tr.spiking_rows])
            if res.halt != nat.SNP_RUNNING:
                break
        reason = HaltReason.STEP_LIMIT if res.halt == nat.SNP_HALT_STEP_LIMIT else HaltReason.NO_APPLICABLE_RULES
        return Trace(configs=configs, halt_reason=reason,
                     delays=delays if want_d else None, spiking=spiking if want_s else None)

    def trace_digests(self, options: SimOptions, initial: np.ndarray | None = None,
                      rows_per_call: int = 1 << 16) -> "TraceDigests":
        """``trace`` with the rows kept on the device: one 64-bit digest per
        recorded row (``row_digest``) comes back instead of the row."""
        flags = _REC_FLAGS[options.record] | nat.SNP_REC_DIGEST
        self.begin(initial)
        opts = self._opts(options.max_steps, options.selection, record=flags)
        out = {"c": [], "d": [], "s": []}
        res = nat.Result()
        while True:
            cap = rows_per_call
            bufs = {k: np.zeros(cap, dtype=np.uint64) for k in out}
            tr = nat.TraceOut()
            tr.cap = cap
            tr.config_digests, tr.delay_digests, tr.spiking_digests = (nat.ptr(bufs[k]) for k in ("c", "d", "s"))
            rc = self._lib.snp_advance(self._h, nat.ctypes.byref(opts), cap, nat.ctypes.byref(tr), nat.ctypes.byref(res))
            if rc:
                self._raise(rc, res)
            out["c"].append(bufs["c"][: tr.config_rows])
            out["d"].append(bufs["d"][: tr.config_rows])
            out["s"].append(bufs["s"][: tr.spiking_rows])
            if res.halt != nat.SNP_RUNNING:
                break
        reason = HaltReason.STEP_LIMIT if res.halt == nat.SNP_HALT_STEP_LIMIT else HaltReason.NO_APPLICABLE_RULES
        cat = {k: np.concatenate(v) for k, v in out.items()}
        return TraceDigests(cat["c"], cat["d"] if flags & nat.SNP_REC_DELAYS else None,
                            cat["s"] if flags & nat.SNP_REC_SPIKING else None, reason)

    def run_final(self, max_steps: int, selection: Selection = FirstApplicable(),
                  initial: np.ndarray | None = None, collect_stats: bool = False,
                  want_delays: bool = True) -> "RunResult":
        """Run to halt on the device; return only the final state."""
        q = self.q
        cfg = np.empty(q, dtype=np.int64)
        dly = np.empty(q, dtype=np.int64) if want_delays else None
        opts = self._opts(max_steps, selection, collect_stats=collect_stats)
        res = nat.Result()
        arr = None if initial is None else _c64(initial)
        rc = self._lib.snp_run(self._h, nat.ptr(arr), nat.ctypes.byref(opts), nat.ptr(cfg), nat.ptr(dly),
                               nat.ctypes.byref(res))
        if rc:
            self._raise(rc, res)
        reason = HaltReason.STEP_LIMIT if res.halt == nat.SNP_HALT_STEP_LIMIT else HaltReason.NO_APPLICABLE_RULES
        return RunResult(cfg, dly, int(res.steps), reason, res.stats_dict(), int(res.kernel_launches),
                         float(self._lib.snp_last_device_ms(self._h)))

    def run_device(self, max_steps: int, initial, final_config, selection: Selection = FirstApplicable(),
                   final_delays=None) -> nat.Result:
        """snp_run with device-resident buffers: ``initial`` / ``final_config`` /
        ``final_delays`` are int64 CUDA tensors of q elements (anything with
        ``data_ptr()``); the copies are device-to-device on the engine's
        stream (no PCIe)."""
        for t in (initial, final_config) + (() if final_delays is None else (final_delays,)):
            if t.numel() != self.q or str(t.dtype) != "torch.int64" or not t.is_cuda or not t.is_contiguous():
                raise ValueError("run_device needs contiguous int64 CUDA tensors of q elements")
        opts = self._opts(max_steps, selection)
        res = nat.Result()
        vp = nat.ctypes.c_void_p
        rc = self._lib.snp_run(self._h, vp(initial.data_ptr()), nat.ctypes.byref(opts), vp(final_config.data_ptr()),
                               None if final_delays is None else vp(final_delays.data_ptr()), nat.ctypes.byref(res))
        if rc:
            self._raise(rc, res)
        return res

    def time_steps(self, steps: int, selection: Selection = FirstApplicable(), per_kernel: bool = False,
                   collect_stats: bool = False) -> tuple[float, float, nat.Result]:
        """Device-timed segment of ``steps`` steps from the current state."""
        opts = self._opts(1 << 62, selection, collect_stats=collect_stats)
        total = nat.ctypes.c_double()
        kern = nat.ctypes.c_double()
        res = nat.Result()
        rc = self._lib.snp_time_steps(self._h, nat.ctypes.byref(opts), int(steps), nat.ctypes.byref(total),
                                      nat.ctypes.byref(kern) if per_kernel else None, nat.ctypes.byref(res))
        if rc:
            self._raise(rc, res)
        return total.value, (kern.value if per_kernel else float("nan")), res

    # -- externally exchanged stepping (row partition, sharded.py) ------------------

    def exchange_info(self) -> nat.Exchange:
        x = nat.Exchange()
        nat.check(self._lib.snp_exchange_info(self._h, nat.ctypes.byref(x)))
        return x

    def set_stream(self, stream_ptr: int | None) -> None:
        nat.check(self._lib.snp_set_stream(self._h, nat.ctypes.c_void_p(stream_ptr or 0)))

    def configure(self, max_steps: int, selection: Selection, collect_stats: bool = False, record: int = 0) -> None:
        """Run parameters for launch_step; ``record`` (SNP_REC_* flags) keeps
        every row of the run on the device for read_trace."""
        opts = self._opts(max_steps, selection, record=int(record), collect_stats=collect_stats)
        rc = self._lib.snp_configure(self._h, nat.ctypes.byref(opts))
        if rc:
            self._raise(rc)

    def read_trace(self, n_configs: int, n_spiking: int, record: int):
        """Rows 0..n_configs-1 (configs / delays) and 0..n_spiking-1 (chosen,
        this engine's rule indices or -1) of a recording run."""
        q = self.q
        cfg = np.empty((n_configs, q), np.int64) if record & nat.SNP_REC_CONFIGS else None
        dly = np.empty((n_configs, q), np.int64) if record & nat.SNP_REC_DELAYS else None
        ch = np.empty((n_spiking, q), np.int64) if record & nat.SNP_REC_SPIKING else None
        rc = self._lib.snp_read_trace(self._h, 0, n_configs, nat.ptr(cfg), nat.ptr(dly), None)
        if rc:
            self._raise(rc)
        if ch is not None and n_spiking:
            rc = self._lib.snp_read_trace(self._h, 0, n_spiking, None, None, nat.ptr(ch))
            if rc:
                self._raise(rc)
        return cfg, dly, ch

    def layout_digest(self) -> tuple[int, ...]:
        """Digests of the tiled layout arrays (snp_engine_layout_digest)."""
        out = np.zeros(6, dtype=np.uint64)
        nat.check(self._lib.snp_engine_layout_digest(self._h, nat.ptr(out)))
        return tuple(int(x) for x in out)

    def ipc_handle(self) -> bytes:
        buf = nat.ctypes.create_string_buffer(nat.SNP_IPC_HANDLE_BYTES)
        nat.check(self._lib.snp_exchange_ipc_handle(self._h, buf))
        return buf.raw

    def connect_peers(self, handles: list[bytes]) -> None:
        blob = b"".join(handles)
        if len(blob) != nat.SNP_IPC_HANDLE_BYTES * len(handles):
            raise ValueError("IPC handles must be SNP_IPC_HANDLE_BYTES each")
        nat.check(self._lib.snp_exchange_connect(self._h, blob, len(handles)))

    @staticmethod
    def connect_local(engines: list["DeviceEngine"]) -> None:
        arr = (nat.ctypes.c_void_p * len(engines))(*[e._h for e in engines])
        nat.check(nat.load().snp_exchange_connect_local(arr, len(engines)))

    def launch_step(self) -> None:
        rc = self._lib.snp_launch_step(self._h)
        if rc:
            self._raise(rc)

    def poll(self) -> nat.Result:
        res = nat.Result()
        rc = self._lib.snp_poll(self._h, nat.ctypes.byref(res))
        if rc:
            self._raise(rc, res)
        return res

    def read_state(self) -> tuple[np.ndarray, np.ndarray]:
        cfg = np.empty(self.q, dtype=np.int64)
        dly = np.empty(self.q, dtype=np.int64)
        rc = self._lib.snp_read_state(self._h, nat.ptr(cfg), nat.ptr(dly))
        if rc:
            self._raise(rc)
        return cfg, dly

    # -- phase functions ----------------------------------------------------------

    def sv_calc(self, config, delays, selection: Selection, step: int) -> np.ndarray:
        policy, seed = policy_code(selection)
        cfg, dly = _c64(config), _c64(delays)
        out = np.empty(self.q, dtype=np.int64)
        rc = self._lib.snp_sv_calc(self._h, nat.ptr(cfg), nat.ptr(dly), policy, seed, int(step), nat.ptr(out))
        if rc:
            self._raise(rc)
        return out

    def step(self, config, delays, chosen, row_visits: np.ndarray | None = None) -> np.ndarray:
        cfg, dly, ch = _c64(config), _c64(delays), _c64(chosen)
        out = np.empty(self.q, dtype=np.int64)
        visits = None
        if row_visits is not None:
            visits = _c64(row_visits)
        rc = self._lib.snp_step(self._h, nat.ptr(cfg), nat.ptr(dly), nat.ptr(ch), nat.ptr(out), nat.ptr(visits))
        if rc:
            self._raise(rc)
        if row_visits is not None and visits is not row_visits:
            row_visits[...] = visits
        return out

    def update_delays(self, delays, chosen) -> np.ndarray:
        dly, ch = _c64(delays), _c64(chosen)
        out = np.empty(self.q, dtype=np.int64)
        rc = self._lib.snp_update_delays(self._h, nat.ptr(dly), nat.ptr(ch), nat.ptr(out))
        if rc:
            self._raise(rc)
        return out


@dataclass(frozen=True)
class RunResult:
    """Final state of a device run (extension; no per-step trace)."""

    config: np.ndarray
    delays: np.ndarray | None
    steps: int
    halt_reason: HaltReason
    stats: dict
    kernel_launches: int
    device_ms: float


# -- reference API --------------------------------------------------------------

class Prepared:
    """A system compiled for one backend (engine.py:377-385).

    ``rules``/``rule_map`` are the host rule vector and offsets; ``matrix``
    (the reference's host layout of ``fmt``) is built on first access only;
    ``engine`` holds the device layouts.
    """

    def __init__(self, system, fmt: Format, rules: RuleVector, rule_map: NeuronRuleMap,
                 engine: DeviceEngine, arrays: SystemArrays):
        self.system = system
        self.fmt = fmt
        self.rules = rules
        self.rule_map = rule_map
        self.engine = engine
        self.arrays = arrays
        self._matrix = None

    @property
    def matrix(self):
        if self._matrix is None:
            a = self.arrays
            q = a.neuron_count
            if self.fmt is Format.SPARSE:
                self._matrix = sparse_from_arrays(q, a.rules, a.adj_offsets, a.adj_targets)
            elif self.fmt is Format.ELL:
                self._matrix = ell_from_arrays(q, a.rules, a.adj_offsets, a.adj_targets)
            else:
                self._matrix = compressed_from_arrays(q, a.adj_offsets, a.adj_targets)
        return self._matrix


def prepare(system: SNPSystem | SystemArrays, fmt: Format, variant: str = "auto",
            device: int = 0) -> Prepared:
    """Build the device structures ``fmt`` needs (time it apart from runs)."""
    fmt = Format(fmt)
    if fmt is Format.ORACLE:
        raise ValueError("Format.ORACLE is the reference's CPU interpreter; in this package it is "
                         "test infrastructure (oracle/), not a simulation backend")
    arrays = system_arrays(system)
    eng = DeviceEngine(fmt, arrays.neuron_count, arrays.rules, arrays.rule_map.offsets, arrays.initial,
                       adj=(arrays.adj_offsets, arrays.adj_targets), variant=variant, device=device)
    return Prepared(system, fmt, arrays.rules, arrays.rule_map, eng, arrays)


def simulate(system, fmt: Format, options: SimOptions) -> Trace:
    return simulate_prepared(prepare(system, fmt), options)


def simulate_prepared(prep: Prepared, options: SimOptions) -> Trace:
    return prep.engine.trace(options)


@dataclass(frozen=True)
class TraceDigests:
    """Per-row digests of a recorded run (``row_digest`` of ``configs[k]``,
    ``delays[k]``, ``spiking[k]``); extension for runs too large to copy."""

    configs: np.ndarray
    delays: np.ndarray | None
    spiking: np.ndarray | None
    halt_reason: HaltReason

    @property
    def steps(self) -> int:
        return len(self.configs) - 1


_DIG_A, _DIG_B = np.uint64(0x9E3779B97F4A7C15), np.uint64(0xD6E8FEB86659FD93)


def row_digest(row) -> int:
    """Digest of one trace row (include/snpb200.h SNP_REC_DIGEST): the sum
    over j of fmix64(v_j * A + (j + 1) * B) mod 2^64."""
    v = np.asarray(row, dtype=np.int64).astype(np.uint64)
    j = np.arange(1, v.size + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = v * _DIG_A + j * _DIG_B
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return int(z.sum(dtype=np.uint64))


def trace_digests(prep: Prepared, options: SimOptions) -> TraceDigests:
    """``simulate_prepared`` with every recorded row reduced to a 64-bit
    digest on the device (8 bytes per row cross PCIe instead of 8q)."""
    return prep.engine.trace_digests(options)


def run_final(prep: Prepared, options: SimOptions, collect_stats: bool = False) -> RunResult:
    """Extension: the run of ``simulate_prepared`` without the per-step trace."""
    return prep.engine.run_final(options.max_steps, options.selection, collect_stats=collect_stats)


# -- phase functions (engine.py:192-366) --------------------------------------------

_PHASE_CACHE: OrderedDict = OrderedDict()
_PHASE_CACHE_MAX = 16


def _content_key(*arrays) -> str:
    """Digest of the arrays' contents (shape, dtype, bytes): an engine built
    from them is reused only while the inputs are unchanged, so in-place
    edits between calls are seen, as in the reference (which recomputes
    from the current arrays every call)."""
    import hashlib
    h = hashlib.blake2b(digest_size=16)
    for x in arrays:
        x = np.ascontiguousarray(x)
        h.update(repr((x.shape, x.dtype.str)).encode())
        if x.size:
            h.update(memoryview(x).cast("B"))
    return h.hexdigest()


def _rule_arrays(rules: RuleVector) -> tuple:
    return (rules.threshold, rules.is_exact, rules.consumed, rules.produced, rules.delay, rules.neuron)


def _phase_engine(key, build):
    """Engines for the phase functions, cached by the content of their inputs
    (at most ``_PHASE_CACHE_MAX``; ``clear_phase_cache`` frees them)."""
    hit = _PHASE_CACHE.get(key)
    if hit is not None:
        _PHASE_CACHE.move_to_end(key)
        return hit
    eng = build()
    _PHASE_CACHE[key] = eng
    while len(_PHASE_CACHE) > _PHASE_CACHE_MAX:
        _PHASE_CACHE.popitem(last=False)
    return eng


def clear_phase_cache() -> None:
    """Drop the device engines cached by the phase functions (frees their
    device memory)."""
    _PHASE_CACHE.clear()


def _selection_engine(rules: RuleVector, q: int, offsets: np.ndarray | None = None) -> DeviceEngine:
    off = offsets if offsets is not None else offsets_from_owners(np.asarray(rules.neuron), q)

    def build():
        empty = (np.zeros(q + 1, dtype=np.int64), np.zeros(0, dtype=np.int64))
        return DeviceEngine(Format.COMPRESSED, q, rules, off, adj=empty)
    return _phase_engine(("sel", q, _content_key(*_rule_arrays(rules), off)), build)


def sv_calc(config: np.ndarray, delays: np.ndarray, rules: RuleVector, rule_map: NeuronRuleMap,
            selection: Selection, step: int = 0, workers: int = 1) -> SpikingVector:
    q = int(np.asarray(config).shape[0])
    eng = _selection_engine(rules, q, rule_map.offsets)
    return SpikingVector(eng.sv_calc(config, delays, selection, step))


def _matrix_engine(fmt: Format, matrix, rules: RuleVector, q: int) -> DeviceEngine:
    def build():
        off = offsets_from_owners(np.asarray(rules.neuron), q)
        kw = {"syn": matrix} if fmt is Format.COMPRESSED else (
            {"ell": matrix} if fmt is Format.ELL else {"sparse": matrix})
        return DeviceEngine(fmt, q, rules, off, **kw)
    if fmt is Format.COMPRESSED:
        mats = (matrix.target,)
    elif fmt is Format.ELL:
        mats = (matrix.target, matrix.amount)
    else:
        mats = (matrix.data,)
    return _phase_engine((fmt, q, _content_key(*mats, *_rule_arrays(rules))), build)


def _step(fmt: Format, state: SimState, matrix, rules: RuleVector, row_visits=None) -> np.ndarray:
    q = int(np.asarray(state.config).shape[0])
    eng = _matrix_engine(fmt, matrix, rules, q)
    return eng.step(state.config, state.delays, state.spiking.chosen, row_visits)


def step_sparse(state: SimState, matrix: SparseMatrix, rules: RuleVector, workers: int = 1) -> np.ndarray:
    return _step(Format.SPARSE, state, matrix, rules)


def step_ell(state: SimState, matrix: EllMatrix, rules: RuleVector, workers: int = 1,
             row_visits: np.ndarray | None = None) -> np.ndarray:
    return _step(Format.ELL, state, matrix, rules, row_visits)


def step_compressed(state: SimState, matrix: SynapseMatrix, rules: RuleVector,
                    workers: int = 1) -> np.ndarray:
    return _step(Format.COMPRESSED, state, matrix, rules)


def update_delays(delays: np.ndarray, spiking: SpikingVector, rules: RuleVector) -> np.ndarray:
    q = int(np.asarray(delays).shape[0])
    return _selection_engine(rules, q).update_delays(delays, spiking.chosen)
