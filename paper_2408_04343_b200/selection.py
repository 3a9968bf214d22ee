"""Rule-selection policies (drop-in for ``snpsim.selection``).

Reference: ``pkg/src/snpsim/selection.py``.

* ``FirstApplicable``   -- lowest-index applicable rule (selection.py:21-23)
* ``SeededRandom(seed)`` -- the ``mix64(seed, step, neuron) % count``-th
  applicable rule in index order (selection.py:26-31, 65-71)
* ``mix64``              -- SplitMix64-style finaliser over (seed, step,
  neuron) mod 2**64 (selection.py:37-45)

The simulation itself never calls these Python helpers: the B200 kernels
evaluate the same hash on device (``csrc/snp_device.cuh``, ``mix64``).
They are kept because the reference exports them and its tests pin the
vectorised form against the scalar one (test_engine.py:52-58).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
MIX_M1 = 0xBF58476D1CE4E5B9
MIX_M2 = 0x94D049BB133111EB


@dataclass(frozen=True)
class FirstApplicable:
    """The lowest-index applicable rule of each open neuron fires."""


@dataclass(frozen=True)
class SeededRandom:
    """Uniform pick among applicable rules keyed by (seed, step, neuron)."""

    seed: int


Selection = FirstApplicable | SeededRandom


def _finalize(z: int) -> int:
    z ^= z >> 30
    z = (z * MIX_M1) & MASK64
    z ^= z >> 27
    z = (z * MIX_M2) & MASK64
    return z ^ (z >> 31)


def mix64(seed: int, step: int, neuron: int) -> int:
    start = (seed + GOLDEN_GAMMA * (step + 1) + MIX_M1 * (neuron + 1)) & MASK64
    return _finalize(start)


def mix64_array(seed: int, step: int, neurons: np.ndarray) -> np.ndarray:
    """Vectorised :func:`mix64` in wrapping uint64 arithmetic."""
    base = np.uint64((seed + GOLDEN_GAMMA * (step + 1)) & MASK64)
    with np.errstate(over="ignore"):
        z = base + np.uint64(MIX_M1) * (np.asarray(neurons, dtype=np.uint64) + np.uint64(1))
        z = z ^ (z >> np.uint64(30))
        z = z * np.uint64(MIX_M1)
        z = z ^ (z >> np.uint64(27))
        z = z * np.uint64(MIX_M2)
        z = z ^ (z >> np.uint64(31))
    return z


def choose_index(selection: Selection, step: int, neuron: int, count: int) -> int:
    if count <= 0:
        raise ValueError("choose_index needs at least one applicable rule")
    if isinstance(selection, SeededRandom):
        return mix64(selection.seed, step, neuron) % count
    return 0


def policy_code(selection: Selection) -> tuple[int, int]:
    """``(policy, seed mod 2**64)`` as passed through the C ABI
    (``SNP_POLICY_FIRST`` = 0, ``SNP_POLICY_SEEDED`` = 1)."""
    if isinstance(selection, SeededRandom):
        return 1, int(selection.seed) & MASK64
    if isinstance(selection, FirstApplicable):
        return 0, 0
    raise TypeError(f"unknown selection policy {selection!r}")
