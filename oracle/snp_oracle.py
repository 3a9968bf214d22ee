"""CPU ORACLE -- test infrastructure only (never the product path).

Restatement of the reference ``snpsim`` 0.1.0 semantics for one SNP
transition step and the run loop, used as the parity checker of the B200
engine and as the CPU baseline of ``bench.py``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / --impl
reference) may import this module.

Three restatements, each citing the reference (``/root/reference/pkg/src/
snpsim``) line it follows:

* :func:`interpret` -- the per-neuron sequential interpreter of
  ``oracle.py:21-101`` (Python ints; no matrices).
* :class:`VectorEngine` -- the vectorised numpy engine of ``engine.py:192-461``
  (sv_calc with searchsorted, np.add.at scatters, chunked thread pool).  This
  is the "port" timed as the reference CPU arm.
* :mod:`oracle.coracle` -- the same interpreter in C (``snp_oracle.c``) for
  full-size parity (10^7 neurons in seconds).

Pinned against the reference itself: ``tests/golden/make_golden.py`` runs the
reference package in the build container and commits its outputs (Tables
1-3, mix64 KATs, traces / digests of the sort family, delay scenarios, 1000
random systems x 2 policies, synth-v1 traces); ``tests/test_oracle_golden.py``
checks all three restatements against those fixtures.  Parity: pinned.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

MASK64 = (1 << 64) - 1
_G = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB

HALT_STEP_LIMIT = "step_limit"
HALT_NO_APPLICABLE = "no_applicable_rules"


class OracleNegative(Exception):
    """NegativeSpikes of the reference (engine.py:48-54, oracle.py:52-56)."""


def mix64(seed: int, step: int, neuron: int) -> int:
    """selection.py:37-45."""
    z = (seed + _G * (step + 1) + _M1 * (neuron + 1)) & MASK64
    z ^= z >> 30
    z = (z * _M1) & MASK64
    z ^= z >> 27
    z = (z * _M2) & MASK64
    return z ^ (z >> 31)


def mix64_vec(seed: int, step: int, neurons: np.ndarray) -> np.ndarray:
    """selection.py:48-62 (uint64 wraparound)."""
    base = np.uint64((seed + _G * (step + 1)) & MASK64)
    with np.errstate(over="ignore"):
        z = base + np.uint64(_M1) * (np.asarray(neurons, dtype=np.uint64) + np.uint64(1))
        z ^= z >> np.uint64(30)
        z *= np.uint64(_M1)
        z ^= z >> np.uint64(27)
        z *= np.uint64(_M2)
        z ^= z >> np.uint64(31)
    return z


@dataclass
class OracleSystem:
    """Plain arrays: rule vector grouped by neuron (matrices.py:48-73) plus
    the out-adjacency (ascending targets, model.py:255-257)."""

    initial: np.ndarray     # int64[q]
    offsets: np.ndarray     # int64[q+1]
    threshold: np.ndarray   # int64[m]
    is_exact: np.ndarray    # bool[m]
    consumed: np.ndarray    # int64[m]
    produced: np.ndarray    # int64[m]
    delay: np.ndarray       # int64[m]
    adj_offsets: np.ndarray  # int64[q+1]
    adj_targets: np.ndarray  # int64[S]

    @property
    def q(self) -> int:
        return int(self.initial.shape[0])

    @property
    def m(self) -> int:
        return int(self.threshold.shape[0])

    @classmethod
    def from_arrays(cls, arrays) -> "OracleSystem":
        """From anything shaped like ``SystemArrays`` (initial, rules,
        rule_map, adj_offsets, adj_targets)."""
        r = arrays.rules
        c = lambda a: np.ascontiguousarray(a, dtype=np.int64)
        return cls(c(arrays.initial), c(arrays.rule_map.offsets), c(r.threshold),
                   np.ascontiguousarray(r.is_exact, dtype=bool), c(r.consumed), c(r.produced),
                   c(r.delay), c(arrays.adj_offsets), c(arrays.adj_targets))

    @classmethod
    def from_npz(cls, data, prefix: str = "") -> "OracleSystem":
        g = lambda k: np.asarray(data[prefix + k])
        return cls(g("initial").astype(np.int64), g("offsets").astype(np.int64),
                   g("threshold").astype(np.int64), g("is_exact").astype(bool),
                   g("consumed").astype(np.int64), g("produced").astype(np.int64),
                   g("delay").astype(np.int64), g("adj_offsets").astype(np.int64),
                   g("adj_targets").astype(np.int64))

    def to_npz_dict(self, prefix: str = "") -> dict:
        return {prefix + k: getattr(self, k) for k in (
            "initial", "offsets", "threshold", "is_exact", "consumed", "produced", "delay",
            "adj_offsets", "adj_targets")}

    def owner(self) -> np.ndarray:
        return np.repeat(np.arange(self.q, dtype=np.int64), np.diff(self.offsets))


@dataclass
class OracleTrace:
    configs: list
    halt: str
    delays: list | None = None
    spiking: list | None = None

    @property
    def steps(self) -> int:
        return len(self.configs) - 1


# -- (1) per-neuron interpreter: oracle.py:21-101 -------------------------------------

def interpret_step(s: OracleSystem, config: list[int], delays: list[int], policy: int,
                   seed: int, step: int) -> tuple[list[int], list[int], dict[int, int]]:
    """oracle.py:21-62: scan each open neuron's rules, pick one, apply."""
    q = s.q
    off = s.offsets.tolist()
    thr = s.threshold.tolist()
    exact = s.is_exact.tolist()
    fired: dict[int, int] = {}
    for n in range(q):
        if delays[n] != 0:
            continue
        cnt = config[n]
        ok = [r for r in range(off[n], off[n + 1])
              if (cnt == thr[r] if exact[r] else cnt >= thr[r])]   # model.py:58-61
        if ok:
            k = 0 if policy == 0 else mix64(seed, step, n) % len(ok)  # selection.py:65-71
            fired[n] = ok[k]
    nxt = list(config)
    aoff = s.adj_offsets.tolist()
    adst = s.adj_targets.tolist()
    for n, r in fired.items():
        nxt[n] -= int(s.consumed[r])
        p = int(s.produced[r])
        if p:
            for t in adst[aoff[n]:aoff[n + 1]]:
                if delays[t] == 0:
                    nxt[t] += p
    for n, v in enumerate(nxt):
        if v < 0:
            raise OracleNegative(f"spike count of neuron {n} went negative ({v})")
    nd = [d - 1 if d > 0 else 0 for d in delays]
    for n, r in fired.items():
        nd[n] = int(s.delay[r])
    return nxt, nd, fired


def interpret(s: OracleSystem, max_steps: int, policy: int = 0, seed: int = 0,
              record: str = "full") -> OracleTrace:
    """oracle.py:65-101: same loop and halting contract as engine.py:441-458."""
    q = s.q
    config = [int(v) for v in s.initial]
    delays = [0] * q
    configs = [np.asarray(config, dtype=np.int64)]
    dlog = [np.zeros(q, dtype=np.int64)] if record != "configs" else None
    slog = [] if record == "full" else None
    step = 0
    while True:
        if step == max_steps:
            halt = HALT_STEP_LIMIT
            break
        nxt, nd, fired = interpret_step(s, config, delays, policy, seed, step)
        if not fired and not any(delays):
            halt = HALT_NO_APPLICABLE
            break
        config, delays = nxt, nd
        step += 1
        configs.append(np.asarray(config, dtype=np.int64))
        if dlog is not None:
            dlog.append(np.asarray(delays, dtype=np.int64))
        if slog is not None:
            ch = np.full(q, -1, dtype=np.int64)
            for n, r in fired.items():
                ch[n] = r
            slog.append(ch)
    return OracleTrace(configs, halt, dlog, slog)


# -- (2) vectorised engine: engine.py:170-461 --------------------------------------

def _bounds(total: int, workers: int) -> list[tuple[int, int]]:
    """engine.py:168-179: contiguous near-equal chunks."""
    parts = max(1, min(workers, total))
    base, extra = divmod(total, parts)
    out, lo = [], 0
    for i in range(parts):
        hi = lo + base + (1 if i < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


class VectorEngine:
    """The reference's numpy engine (one format), restated.

    ``fmt`` in {"sparse", "ell", "compressed"}; the layouts are the
    reference's (matrices.py:143-187): dense ``int64[m, q]``, ELL
    ``(target, amount) int64[z+1, m]``, synapse ``int64[z, q]``.
    """

    def __init__(self, s: OracleSystem, fmt: str = "compressed", workers: int = 1,
                 pool: ThreadPoolExecutor | None = None):
        self.s = s
        self.fmt = fmt
        self.workers = workers
        self.owner = s.owner()
        self._pool = pool
        q, m = s.q, s.m
        deg = np.diff(s.adj_offsets)
        z = int(deg.max()) if deg.size else 0
        src = np.repeat(np.arange(q, dtype=np.int64), deg)
        rank = np.arange(s.adj_targets.size, dtype=np.int64) - np.repeat(s.adj_offsets[:-1], deg)
        # vectorised builders equivalent to matrices.py:143-187
        send = np.flatnonzero(s.produced > 0)
        per = deg[self.owner[send]]
        r_idx = np.repeat(send, per)
        within = np.arange(int(per.sum()), dtype=np.int64) - np.repeat(np.cumsum(per) - per, per)
        dst = s.adj_targets[np.repeat(s.adj_offsets[self.owner[send]], per) + within]
        if fmt == "compressed":
            syn = np.full((z, q), -1, dtype=np.int64)
            syn[rank, src] = s.adj_targets
            self.syn = syn
        elif fmt == "ell":
            tgt = np.full((z + 1, m), -1, dtype=np.int64)
            amt = np.zeros((z + 1, m), dtype=np.int64)
            tgt[0] = self.owner
            amt[0] = -s.consumed
            tgt[within + 1, r_idx] = dst
            amt[within + 1, r_idx] = s.produced[r_idx]
            self.ell_t, self.ell_a = tgt, amt
        elif fmt == "sparse":
            dense = np.zeros((m, q), dtype=np.int64)
            dense[r_idx, dst] = s.produced[r_idx]
            dense[np.arange(m), self.owner] = -s.consumed
            self.dense = dense
        else:
            raise ValueError(fmt)

    def _map(self, total: int, fn):
        b = _bounds(total, self.workers)
        if len(b) == 1:
            return [fn(*b[0])]
        if self._pool is None:
            self._pool = ThreadPoolExecutor(max_workers=self.workers)
        return list(self._pool.map(lambda x: fn(*x), b))

    def sv_calc(self, config, delays, policy: int, seed: int, step: int) -> np.ndarray:
        """engine.py:192-236."""
        s = self.s
        off = s.offsets

        def chunk(lo, hi):
            chosen = np.full(hi - lo, -1, dtype=np.int64)
            r0, r1 = int(off[lo]), int(off[hi])
            if r0 == r1:
                return chosen
            own = self.owner[r0:r1]
            cnt = config[own]
            thr = s.threshold[r0:r1]
            ok = (delays[own] == 0) & np.where(s.is_exact[r0:r1], cnt == thr, cnt >= thr)
            idx = np.flatnonzero(ok)
            if idx.size == 0:
                return chosen
            owners = own[idx]
            neurons = np.unique(owners)
            first = np.searchsorted(owners, neurons, side="left")
            if policy == 0:
                pick = first
            else:
                per = np.searchsorted(owners, neurons, side="right") - first
                pick = first + (mix64_vec(seed, step, neurons) % per.astype(np.uint64)).astype(np.int64)
            chosen[neurons - lo] = idx[pick] + r0
            return chosen

        parts = self._map(s.q, chunk)
        return parts[0] if len(parts) == 1 else np.concatenate(parts)

    def step(self, config, delays, chosen) -> np.ndarray:
        if self.fmt == "compressed":
            return self._step_compressed(config, delays, chosen)
        if self.fmt == "ell":
            return self._step_ell(config, delays, chosen)
        return self._step_sparse(config, delays, chosen)

    def _step_sparse(self, config, delays, chosen):
        """engine.py:239-266."""
        flags = np.zeros(self.s.m, dtype=np.uint8)
        flags[chosen[chosen >= 0]] = 1
        active = np.flatnonzero(flags)
        if active.size:
            active = active[delays[self.owner[active]] == 0]
        rows = self.dense[active]
        parts = self._map(config.shape[0], lambda lo, hi: rows[:, lo:hi].sum(axis=0, dtype=np.int64))
        delta = parts[0] if len(parts) == 1 else np.concatenate(parts)
        nxt = np.where(delays == 0, config + delta, config)
        if (nxt < 0).any():
            raise OracleNegative("negative")
        return nxt

    def _step_ell(self, config, delays, chosen):
        """engine.py:269-310."""
        flags = np.zeros(self.s.m, dtype=np.uint8)
        flags[chosen[chosen >= 0]] = 1
        active = np.flatnonzero(flags)
        if active.size:
            active = active[delays[self.owner[active]] == 0]
        q = config.shape[0]
        rows = self.ell_t.shape[0]

        def chunk(lo, hi):
            delta = np.zeros(q, dtype=np.int64)
            alive = active[lo:hi]
            row = 0
            while alive.size and row < rows:
                tgt = self.ell_t[row, alive]
                amt = self.ell_a[row, alive]
                live = tgt >= 0
                tgt, amt = tgt[live], amt[live]
                op = delays[tgt] == 0
                np.add.at(delta, tgt[op], amt[op])
                alive = alive[live]
                row += 1
            return delta

        delta = sum(self._map(active.size, chunk))
        nxt = config + delta
        if (nxt < 0).any():
            raise OracleNegative("negative")
        return nxt

    def _step_compressed(self, config, delays, chosen):
        """engine.py:313-355."""
        firing = np.flatnonzero(chosen >= 0)
        if firing.size:
            firing = firing[delays[firing] == 0]
        q = config.shape[0]
        rows = self.syn.shape[0]
        s = self.s

        def chunk(lo, hi):
            delta = np.zeros(q, dtype=np.int64)
            cols = firing[lo:hi]
            rid = chosen[cols]
            delta[cols] -= s.consumed[rid]
            prod = s.produced[rid]
            send = prod > 0
            alive, amounts = cols[send], prod[send]
            row = 0
            while alive.size and row < rows:
                tgt = self.syn[row, alive]
                live = tgt >= 0
                tgt, amt = tgt[live], amounts[live]
                op = delays[tgt] == 0
                np.add.at(delta, tgt[op], amt[op])
                alive, amounts = alive[live], amt
                row += 1
            return delta

        delta = sum(self._map(firing.size, chunk))
        nxt = config + delta
        if (nxt < 0).any():
            raise OracleNegative("negative")
        return nxt

    def update_delays(self, delays, chosen):
        """engine.py:358-366."""
        nxt = np.where(delays > 0, delays - 1, 0)
        fired = chosen >= 0
        if fired.any():
            nxt[fired] = self.s.delay[chosen[fired]]
        return nxt

    def run(self, max_steps: int, policy: int = 0, seed: int = 0, record: str = "configs",
            initial: np.ndarray | None = None) -> OracleTrace:
        """engine.py:416-461."""
        q = self.s.q
        config = np.array(self.s.initial if initial is None else initial, dtype=np.int64)
        delays = np.zeros(q, dtype=np.int64)
        configs = [config.copy()]
        dlog = [delays.copy()] if record in ("configs+delays", "full") else None
        slog = [] if record == "full" else None
        step = 0
        while True:
            if step == max_steps:
                halt = HALT_STEP_LIMIT
                break
            chosen = self.sv_calc(config, delays, policy, seed, step)
            if (chosen < 0).all() and not delays.any():
                halt = HALT_NO_APPLICABLE
                break
            config = self.step(config, delays, chosen)
            delays = self.update_delays(delays, chosen)
            step += 1
            if record != "none":
                configs.append(config.copy())
            if dlog is not None:
                dlog.append(delays.copy())
            if slog is not None:
                slog.append(chosen.copy())
        if record == "none":
            configs.append(config)
        return OracleTrace(configs, halt, dlog, slog)


def trace_digest(configs, delays=None, spiking=None) -> str:
    """sha256 over the int64 rows (configs, then delays, then spiking)."""
    import hashlib
    h = hashlib.sha256()
    for group in (configs, delays, spiking):
        if group is None:
            h.update(b"|none")
            continue
        h.update(b"|%d" % len(group))
        for row in group:
            h.update(np.ascontiguousarray(row, dtype=np.int64).tobytes())
    return h.hexdigest()
