"""Workload families.

Drop-in for ``snpsim.generators`` (reference ``pkg/src/snpsim/generators.py``):
``gen_sort`` (:93-124), ``sort_result`` (:127-131), ``gen_subset_sum``
(:134-183), ``subset_sum_accepted`` (:186-189), ``gen_random`` (:195-230).
``gen_random`` draws from ``random.Random(seed)`` in the same call order as
the reference so the property corpus (tests/conftest.py:11-16 upstream) is
the same set of systems; ``tests/golden`` pins that.

Extensions for scale (no reference counterpart -- SURVEY.md section 8(d)):

* :class:`SystemArrays` -- a validated system held as flat numpy arrays
  (rule vector + offsets + CSR out-adjacency); ``prepare`` accepts it.
* :func:`sort_arrays` -- the ``gen_sort`` system built directly as arrays
  (n=4096 has 16.8M rules; the object builder would need minutes and GBs).
* :func:`synth_v1` -- the counter-based synthetic family used by the bench
  (K3/K4/K5): out-degree exactly 16, 4 rules per neuron.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

import numpy as np

from .matrices import NeuronRuleMap, RuleVector, build_rule_vector, offsets_from_owners
from .model import ModelError, SNPSystem, SystemStats, at_least, exactly
from .selection import mix64_array


class InvalidInstance(ModelError):
    """Instance parameters outside the family's preconditions."""


@dataclass(frozen=True)
class SortInstance:
    """``n`` distinct positive integers (default worst case ``n..1``)."""

    n: int
    values: tuple[int, ...] = ()

    def __post_init__(self):
        if self.n < 1:
            raise InvalidInstance(f"sort instance needs n >= 1, got {self.n}")
        vals = tuple(int(v) for v in (self.values or range(self.n, 0, -1)))
        object.__setattr__(self, "values", vals)
        if len(vals) != self.n:
            raise InvalidInstance(f"expected {self.n} values, got {len(vals)}")
        if min(vals) < 1:
            raise InvalidInstance("sort values must be positive integers")
        if len(set(vals)) != self.n:
            raise InvalidInstance("sort values must be pairwise distinct")


@dataclass(frozen=True)
class SubsetSumInstance:
    values: tuple[int, ...]
    target: int

    def __post_init__(self):
        vals = tuple(int(v) for v in self.values)
        object.__setattr__(self, "values", vals)
        if any(v < 0 for v in vals):
            raise InvalidInstance("subset-sum values must be non-negative")
        if self.target < 0:
            raise InvalidInstance("subset-sum target must be non-negative")
        if self.target > sum(vals):
            raise InvalidInstance(f"target {self.target} exceeds the total {sum(vals)}")

    @classmethod
    def random(cls, n: int, seed: int, low: int = 0, high: int = 50,
               fraction: float = 0.2) -> "SubsetSumInstance":
        if n < 0:
            raise InvalidInstance(f"n must be >= 0, got {n}")
        rng = random.Random(seed)
        vals = tuple(rng.randint(low, high) for _ in range(n))
        k = round(fraction * n)
        return cls(vals, sum(rng.sample(vals, k)) if k else 0)


# -- array-form systems -------------------------------------------------------

@dataclass(frozen=True)
class SystemArrays:
    """A validated system as flat arrays (what the engine consumes).

    ``adj_offsets``/``adj_targets`` is the out-adjacency in CSR form with
    ascending targets per source (the canonical order of model.py:255-257).
    """

    initial: np.ndarray            # int64[q]
    rules: RuleVector
    rule_map: NeuronRuleMap
    adj_offsets: np.ndarray        # int64[q+1]
    adj_targets: np.ndarray        # int64[S]
    output_neuron: int | None = None

    @property
    def neuron_count(self) -> int:
        return int(self.initial.shape[0])

    @property
    def initial_spikes(self) -> np.ndarray:
        return self.initial

    @property
    def rule_count(self) -> int:
        return len(self.rules)

    def out_degrees(self) -> np.ndarray:
        return np.diff(self.adj_offsets)

    def max_out_degree(self) -> int:
        deg = self.out_degrees()
        return int(deg.max()) if deg.size else 0

    def stats(self) -> SystemStats:
        z = self.max_out_degree()
        return SystemStats(self.neuron_count, self.rule_count, z, z + 1, z)

    def ensure_validated(self) -> "SystemArrays":
        return self


def system_arrays(system) -> SystemArrays:
    """Array form of an ``SNPSystem`` (identity for ``SystemArrays``)."""
    if isinstance(system, SystemArrays):
        return system
    system.ensure_validated()
    rules, rule_map = build_rule_vector(system)
    off, dst = system.adjacency_csr()
    return SystemArrays(np.asarray(system.initial_spikes, dtype=np.int64), rules, rule_map,
                        off, dst, system.output_neuron)


# -- families -----------------------------------------------------------------

def gen_sort(instance: SortInstance) -> SNPSystem:
    """Natural-number sorter: inputs ``0..n-1``, detectors ``n..2n-1``,
    outputs ``2n..3n-1``.  Detector ``j`` (1-based) fires on exactly
    ``n+1-j`` spikes; its forgetting rules list the counts above that
    ascending, then the counts below it descending."""
    n = instance.n
    sys_ = SNPSystem()
    ins = [sys_.add_neuron(v) for v in instance.values]
    dets = [sys_.add_neuron(0) for _ in range(n)]
    outs = [sys_.add_neuron(0) for _ in range(n)]
    for i in ins:
        sys_.add_rule(i, at_least(1), 1, 1, 0)
        for d in dets:
            sys_.add_synapse(i, d)
    for j, det in enumerate(dets, start=1):
        fire = n + 1 - j
        sys_.add_rule(det, exactly(fire), fire, 1, 0)
        for k in list(range(fire + 1, n + 1)) + list(range(fire - 1, 0, -1)):
            sys_.add_rule(det, exactly(k), k, 0, 0)
        for o in outs[j - 1:]:
            sys_.add_synapse(det, o)
    return sys_.validate()


def sort_arrays(instance: SortInstance) -> SystemArrays:
    """:func:`gen_sort` built straight into arrays (identical content)."""
    n = instance.n
    q = 3 * n
    init = np.zeros(q, dtype=np.int64)
    init[:n] = instance.values
    # inputs: one rule each; detector j (1-based) owns n rules
    det_j = np.arange(1, n + 1, dtype=np.int64)
    fire = n + 1 - det_j
    # per detector the counts in rule order: fire, fire+1..n, fire-1..1
    k = np.arange(n, dtype=np.int64)[None, :]  # rule slot within detector
    f = fire[:, None]
    above = n - f  # how many counts above fire
    counts = np.where(k == 0, f, np.where(k <= above, f + k, f - (k - above)))
    counts = counts.reshape(-1)
    m = n + n * n
    thr = np.empty(m, dtype=np.int64)
    thr[:n] = 1
    thr[n:] = counts
    exact = np.ones(m, dtype=bool)
    exact[:n] = False
    cons = thr.copy()
    prod = np.zeros(m, dtype=np.int64)
    prod[:n] = 1
    prod[n::n] = 1  # first rule of every detector fires
    owner = np.empty(m, dtype=np.int64)
    owner[:n] = np.arange(n)
    owner[n:] = np.repeat(np.arange(n, 2 * n), n)
    rules = RuleVector(thr, exact, cons, prod, np.zeros(m, dtype=np.int64), owner)
    # adjacency: inputs -> all detectors; detector j -> outputs j-1..n-1
    deg = np.zeros(q, dtype=np.int64)
    deg[:n] = n
    deg[n:2 * n] = n - np.arange(n)
    off = np.zeros(q + 1, dtype=np.int64)
    np.cumsum(deg, out=off[1:])
    in_part = np.tile(np.arange(n, 2 * n, dtype=np.int64), n)
    det_part = np.concatenate([np.arange(2 * n + j, 3 * n, dtype=np.int64) for j in range(n)]) \
        if n else np.zeros(0, dtype=np.int64)
    dst = np.concatenate([in_part, det_part])
    return SystemArrays(init, rules, NeuronRuleMap(offsets_from_owners(owner, q)), off, dst)


def sort_result(trace, n: int) -> list[int]:
    return [int(v) for v in trace.configs[-1][2 * n:3 * n]]


def gen_subset_sum(instance: SubsetSumInstance) -> SNPSystem:
    """Nondeterministic subset-sum: trigger, per value ``v`` stores/chooser/
    relay, adder last (the output neuron)."""
    vals = instance.values
    n = len(vals)
    sys_ = SNPSystem()
    trig = sys_.add_neuron(1)
    sys_.add_rule(trig, at_least(1), 1, 1, 0)
    choosers, relays = [], []
    for v in vals:
        stores = [sys_.add_neuron(1) for _ in range(v)]
        ch = sys_.add_neuron(0)
        rl = sys_.add_neuron(0)
        for s in stores:
            sys_.add_rule(s, at_least(1), 1, 1, 0)
            sys_.add_synapse(s, ch)
        sys_.add_rule(ch, exactly(v + 1), v + 1, v + 1, 0)  # take
        sys_.add_rule(ch, exactly(v + 1), v + 1, 1, 0)      # skip
        sys_.add_rule(rl, exactly(v + 1), v + 1, v + 1, 1)  # relay a take, one-step delay
        sys_.add_rule(rl, exactly(1), 1, 1, 0)              # relay a skip
        sys_.add_synapse(ch, rl)
        choosers.append(ch)
        relays.append(rl)
    adder = sys_.add_neuron(1)
    fire = instance.target + n + 1
    sys_.add_rule(adder, exactly(fire), fire, 1, 0)
    for ch in choosers:
        sys_.add_synapse(trig, ch)
    for rl in relays:
        sys_.add_synapse(rl, adder)
    sys_.output_neuron = adder
    return sys_.validate()


def subset_sum_accepted(trace, system) -> bool:
    return int(trace.configs[-1][system.output_neuron]) == 0


SUBSET_SUM_STEP_BOUND = 6


def gen_random(q_max: int, rules_per_neuron_max: int, out_degree_max: int,
               spikes_max: int, delay_max: int, seed: int) -> SNPSystem:
    """Random valid system; same ``random.Random`` call sequence as the
    reference so a seed names the same system."""
    if min(q_max, rules_per_neuron_max, out_degree_max, spikes_max) < 1:
        raise InvalidInstance("bounds must be >= 1 (delay_max may be 0)")
    if delay_max < 0:
        raise InvalidInstance(f"delay_max must be >= 0, got {delay_max}")
    rng = random.Random(seed)
    sys_ = SNPSystem()
    q = rng.randint(1, q_max)
    for _ in range(q):
        sys_.add_neuron(rng.randint(0, spikes_max))
    for nid in range(q):
        for _ in range(rng.randint(0, rules_per_neuron_max)):
            roll = rng.random()
            if roll < 0.20:
                c = rng.randint(1, spikes_max)
                sys_.add_rule(nid, exactly(c), c, 0, 0)
                continue
            thr = rng.randint(1, spikes_max)
            c = rng.randint(1, thr)
            p = rng.randint(1, c)
            d = rng.randint(0, delay_max)
            sys_.add_rule(nid, exactly(thr) if roll < 0.55 else at_least(thr), c, p, d)
    if q > 1:
        for nid in range(q):
            pool = [i for i in range(q) if i != nid]
            for dst in rng.sample(pool, rng.randint(0, min(out_degree_max, q - 1))):
                sys_.add_synapse(nid, dst)
    return sys_.validate()


# -- synth-v1 --------------------------------------------------

SYNTH_SEED = 240804343
SYNTH_DEGREE = 16


def synth_v1(q: int, seed: int = SYNTH_SEED, with_delays: bool = False) -> SystemArrays:
    """The synthetic family below, generated natively with all host threads
    (``snpio_synth_v1``; identical to :func:`synth_v1_numpy`)."""
    if q < SYNTH_DEGREE + 1:
        raise InvalidInstance(f"synth_v1 needs q >= {SYNTH_DEGREE + 1}, got {q}")
    return synth_v1_native(q, 0, q, seed, with_delays)


def synth_v1_native(q: int, lo: int, hi: int, seed: int = SYNTH_SEED, with_delays: bool = False) -> SystemArrays:
    """Rows [lo, hi) of synth_v1(q) and the CSR over all q sources of the edges
    entering them (include/snpio.h snpio_synth_v1)."""
    import ctypes

    from .modelfile import _check, _io_lib, _ptr
    lib = _io_lib()
    seed_u = ctypes.c_uint64(seed & ((1 << 64) - 1))
    ne = ctypes.c_int64()
    _check(lib.snpio_synth_v1_edges(q, seed_u, lo, hi, ctypes.byref(ne)))
    n, m = hi - lo, 4 * (hi - lo)
    init, off = np.empty(n, np.int64), np.empty(n + 1, np.int64)
    thr, cons, prod, dly = (np.empty(m, np.int64) for _ in range(4))
    exact = np.empty(m, np.bool_)
    aoff, adst = np.empty(q + 1, np.int64), np.empty(ne.value, np.int64)
    _check(lib.snpio_synth_v1(q, seed_u, 1 if with_delays else 0, lo, hi,
                              *map(_ptr, (init, off, thr, exact, cons, prod, dly, aoff, adst))))
    owner = np.repeat(np.arange(n, dtype=np.int64), 4)
    return SystemArrays(init, RuleVector(thr, exact, cons, prod, dly, owner), NeuronRuleMap(off), aoff, adst)


def synth_v1_numpy(q: int, seed: int = SYNTH_SEED, with_delays: bool = False) -> SystemArrays:
    """Counter-based synthetic system: every quantity is ``mix64(seed,
    stream, neuron)`` so any shard can be rebuilt independently.

    * ``init[i] = h0(i) % 8``
    * 16 out-neighbours: ``t_k(i) = (i + 1 + k*W + h_{1+k}(i) % W) mod q``,
      ``W = (q-1)//16`` -- distinct and non-reflexive by construction,
      stored ascending.
    * rules (in order): ``exactly(t0)/a^t0->a`` (t0 in [2,5]),
      ``at_least(t1)/a^c->a`` (t1 in [3,8], c in [1,t1]), forgetting
      ``exactly(t2)`` (t2 in [1,5]), liveness ``at_least(1)/a->a``.
    * with_delays: rules 0, 1 and 3 get ``d = h % 4`` (K4).
    """
    if q < SYNTH_DEGREE + 1:
        raise InvalidInstance(f"synth_v1 needs q >= {SYNTH_DEGREE + 1}, got {q}")
    idx = np.arange(q, dtype=np.int64)

    def h(stream: int) -> np.ndarray:
        return mix64_array(seed, stream, idx)

    init = (h(0) % np.uint64(8)).astype(np.int64)
    width = (q - 1) // SYNTH_DEGREE
    tg = np.empty((q, SYNTH_DEGREE), dtype=np.int64)
    for k in range(SYNTH_DEGREE):
        jitter = (h(1 + k) % np.uint64(width)).astype(np.int64)
        tg[:, k] = (idx + 1 + k * width + jitter) % q
    tg.sort(axis=1)
    t0 = 2 + (h(17) % np.uint64(4)).astype(np.int64)
    t1 = 3 + (h(18) % np.uint64(6)).astype(np.int64)
    c1 = 1 + (h(19) % t1.astype(np.uint64)).astype(np.int64)
    t2 = 1 + (h(20) % np.uint64(5)).astype(np.int64)
    m = 4 * q
    thr = np.empty((q, 4), dtype=np.int64)
    thr[:, 0], thr[:, 1], thr[:, 2], thr[:, 3] = t0, t1, t2, 1
    cons = np.empty((q, 4), dtype=np.int64)
    cons[:, 0], cons[:, 1], cons[:, 2], cons[:, 3] = t0, c1, t2, 1
    prod = np.tile(np.array([1, 1, 0, 1], dtype=np.int64), (q, 1))
    exact = np.tile(np.array([True, False, True, False]), (q, 1))
    dly = np.zeros((q, 4), dtype=np.int64)
    if with_delays:
        for r, stream in ((0, 21), (1, 22), (3, 23)):
            dly[:, r] = (h(stream) % np.uint64(4)).astype(np.int64)
    owner = np.repeat(idx, 4)
    rules = RuleVector(thr.reshape(m), exact.reshape(m), cons.reshape(m),
                       prod.reshape(m), dly.reshape(m), owner)
    offsets = np.arange(0, m + 1, 4, dtype=np.int64)
    adj_off = np.arange(0, SYNTH_DEGREE * q + 1, SYNTH_DEGREE, dtype=np.int64)
    return SystemArrays(init, rules, NeuronRuleMap(offsets), adj_off, tg.reshape(-1))
