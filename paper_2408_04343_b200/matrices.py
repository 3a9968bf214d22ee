"""Rule store, neuron->rule offsets and the three transition layouts.

Drop-in for ``snpsim.matrices`` (reference ``pkg/src/snpsim/matrices.py``):

* ``RuleVector`` (matrices.py:48-65), ``NeuronRuleMap`` (:68-73)
* ``SparseMatrix`` -- dense ``int64[m, q]`` (:76-80, built :143-154)
* ``EllMatrix``    -- ``(target, amount) int64[z+1, m]``, consumption pair in
  row 0, ascending deliveries, ``NULL`` padding (:83-97, built :157-175)
* ``SynapseMatrix`` -- ``target int64[z, q]`` (:100-112, built :178-187)
* ``storage_elements`` / ``storage_bytes`` (:190-221)

These host arrays are the reference's *interchange* layouts: the
``snp_*`` C ABI accepts them verbatim.  The builders here are vectorised
(numpy scatter over the CSR adjacency) instead of per-entry Python loops, so
they stay usable at 10^6-10^7 neurons; the outputs are identical to the
reference builders (pinned by ``tests/test_matrices.py`` against the golden
Tables 1-3).  The B200 engine does not need them at all: it derives its
device layouts (``csrc/snp_engine.cu``, ``build_device_layouts``) straight from
the rule vector plus the CSR adjacency.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .model import SNPSystem

NULL = -1


class Format(str, enum.Enum):
    """Storage format / backend selector (matrices.py:33-45).

    ``OPTIMIZED`` is the paper's name for ``COMPRESSED`` and
    ``DENSE`` the descriptive name of ``SPARSE`` (the uncompressed matrix);
    both are enum aliases, so iteration still yields the four reference
    members.
    """

    SPARSE = "sparse"
    ELL = "ell"
    COMPRESSED = "compressed"
    ORACLE = "oracle"
    OPTIMIZED = "compressed"
    DENSE = "sparse"

    def __str__(self) -> str:  # pragma: no cover - cosmetic
        return self.value


MATRIX_FORMATS = (Format.SPARSE, Format.ELL, Format.COMPRESSED)


@dataclass(frozen=True)
class RuleVector:
    """Per-rule SoA, grouped contiguously (non-decreasing ``neuron``)."""

    threshold: np.ndarray  # int64[m]
    is_exact: np.ndarray   # bool[m]
    consumed: np.ndarray   # int64[m]
    produced: np.ndarray   # int64[m]; 0 for forgetting rules
    delay: np.ndarray      # int64[m]
    neuron: np.ndarray     # int64[m]

    def __len__(self) -> int:
        return int(self.threshold.shape[0])


@dataclass(frozen=True)
class NeuronRuleMap:
    """Rules of neuron ``i`` are ``offsets[i]:offsets[i+1]``."""

    offsets: np.ndarray  # int64[q+1]


@dataclass(frozen=True)
class SparseMatrix:
    data: np.ndarray  # int64[m, q]


@dataclass(frozen=True)
class EllMatrix:
    target: np.ndarray  # int64[z+1, m]
    amount: np.ndarray  # int64[z+1, m]

    @property
    def rows(self) -> int:
        return int(self.target.shape[0])


@dataclass(frozen=True)
class SynapseMatrix:
    target: np.ndarray  # int64[z, q]

    @property
    def rows(self) -> int:
        return int(self.target.shape[0])


def rule_arrays(rules) -> RuleVector:
    """RuleVector of an already-grouped rule list (one pass over objects)."""
    m = len(rules)
    thr = np.fromiter((r.regex.threshold for r in rules), dtype=np.int64, count=m)
    exact = np.fromiter((int(r.regex.kind) for r in rules), dtype=np.int64, count=m) != 0
    cons = np.fromiter((r.consumed for r in rules), dtype=np.int64, count=m)
    prod = np.fromiter((r.produced for r in rules), dtype=np.int64, count=m)
    dly = np.fromiter((r.delay for r in rules), dtype=np.int64, count=m)
    owner = np.fromiter((r.neuron for r in rules), dtype=np.int64, count=m)
    return RuleVector(thr, exact, cons, prod, dly, owner)


def offsets_from_owners(owner: np.ndarray, q: int) -> np.ndarray:
    offsets = np.zeros(q + 1, dtype=np.int64)
    if owner.size:
        np.cumsum(np.bincount(owner, minlength=q), out=offsets[1:])
    return offsets


def build_rule_vector(system: SNPSystem) -> tuple[RuleVector, NeuronRuleMap]:
    system.ensure_validated()
    vec = rule_arrays(system.rules)
    return vec, NeuronRuleMap(offsets_from_owners(vec.neuron, system.neuron_count))


def _csr_rows(adj_off: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(source of each CSR entry, its rank within the source's list)."""
    deg = np.diff(adj_off)
    src = np.repeat(np.arange(deg.size, dtype=np.int64), deg)
    rank = np.arange(int(adj_off[-1]), dtype=np.int64) - np.repeat(adj_off[:-1], deg)
    return src, rank


def sparse_from_arrays(q: int, rules: RuleVector, adj_off: np.ndarray,
                       adj_dst: np.ndarray) -> SparseMatrix:
    m = len(rules)
    data = np.zeros((m, q), dtype=np.int64)
    if m == 0:
        return SparseMatrix(data)
    rows = np.arange(m, dtype=np.int64)
    deg = np.diff(adj_off)
    sending = np.flatnonzero(rules.produced > 0)
    per_rule = deg[rules.neuron[sending]]
    r_idx = np.repeat(sending, per_rule)
    starts = adj_off[rules.neuron[sending]]
    within = np.arange(int(per_rule.sum()), dtype=np.int64) - np.repeat(
        np.cumsum(per_rule) - per_rule, per_rule)
    cols = adj_dst[np.repeat(starts, per_rule) + within]
    data[r_idx, cols] = rules.produced[r_idx]
    data[rows, rules.neuron] = -rules.consumed
    return SparseMatrix(data)


def ell_from_arrays(q: int, rules: RuleVector, adj_off: np.ndarray,
                    adj_dst: np.ndarray) -> EllMatrix:
    m = len(rules)
    deg = np.diff(adj_off)
    z = int(deg.max()) if deg.size else 0
    target = np.full((z + 1, m), NULL, dtype=np.int64)
    amount = np.zeros((z + 1, m), dtype=np.int64)
    if m == 0:
        return EllMatrix(target, amount)
    target[0] = rules.neuron
    amount[0] = -rules.consumed
    sending = np.flatnonzero(rules.produced > 0)
    per_rule = deg[rules.neuron[sending]]
    r_idx = np.repeat(sending, per_rule)
    within = np.arange(int(per_rule.sum()), dtype=np.int64) - np.repeat(
        np.cumsum(per_rule) - per_rule, per_rule)
    src_pos = np.repeat(adj_off[rules.neuron[sending]], per_rule) + within
    target[within + 1, r_idx] = adj_dst[src_pos]
    amount[within + 1, r_idx] = rules.produced[r_idx]
    return EllMatrix(target, amount)


def compressed_from_arrays(q: int, adj_off: np.ndarray, adj_dst: np.ndarray) -> SynapseMatrix:
    deg = np.diff(adj_off)
    z = int(deg.max()) if deg.size else 0
    target = np.full((z, q), NULL, dtype=np.int64)
    if adj_dst.size:
        src, rank = _csr_rows(adj_off)
        target[rank, src] = adj_dst
    return SynapseMatrix(target)


def adjacency_from_synapse_matrix(matrix: SynapseMatrix) -> tuple[np.ndarray, np.ndarray]:
    """CSR out-adjacency of a reference ``SynapseMatrix`` (first NULL ends a
    column, matrices.py:100-112)."""
    tgt = matrix.target
    z, q = tgt.shape
    if z == 0:
        return np.zeros(q + 1, dtype=np.int64), np.zeros(0, dtype=np.int64)
    live = np.cumprod(tgt >= 0, axis=0).astype(bool)  # alive until the first NULL
    deg = live.sum(axis=0)
    off = np.zeros(q + 1, dtype=np.int64)
    np.cumsum(deg, out=off[1:])
    dst = tgt.T[live.T]
    return off, np.ascontiguousarray(dst, dtype=np.int64)


def build_sparse(system: SNPSystem) -> SparseMatrix:
    system.ensure_validated()
    rules, _ = build_rule_vector(system)
    return sparse_from_arrays(system.neuron_count, rules, *system.adjacency_csr())


def build_ell(system: SNPSystem) -> EllMatrix:
    system.ensure_validated()
    rules, _ = build_rule_vector(system)
    return ell_from_arrays(system.neuron_count, rules, *system.adjacency_csr())


def build_compressed(system: SNPSystem) -> SynapseMatrix:
    system.ensure_validated()
    return compressed_from_arrays(system.neuron_count, *system.adjacency_csr())


def element_count(fmt: Format, q: int, m: int, z: int) -> int:
    """Stored-element formulas of matrices.py:190-208."""
    if fmt is Format.SPARSE:
        return m * q + 3 * m + 2 * q + 1
    if fmt is Format.ELL:
        return m * (2 * z + 5) + 2 * q + 1
    if fmt is Format.COMPRESSED:
        return q * (z + 3) + 4 * m + 1
    raise ValueError(f"no storage accounting for format {fmt!r}")


def storage_elements(fmt: Format, system: SNPSystem) -> int:
    stats = system.ensure_validated().stats()
    return element_count(fmt, stats.q, stats.m, stats.max_out_degree)


def storage_bytes(fmt: Format, system: SNPSystem,
                  matrix_width: int = 4, config_width: int = 8) -> int:
    q = system.neuron_count
    return (storage_elements(fmt, system) - q) * matrix_width + q * config_width
