"""Family benchmark harness (drop-in for ``snpsim.bench``,
``pkg/src/snpsim/bench.py:1-106``): timed runs over the model families,
one CSV row per (size, format, repetition), same header and columns.

``wall_ms`` is the host wall time of ``simulate_prepared`` (device loop,
trace copies included, as in the reference); the structure build
(``prepare``: host layout + upload) is timed separately and reported in the
log line only.  ``variant`` selects the COMPRESSED kernel (tiled / pull /
push), an extension with no reference counterpart.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

from .engine import Format, SimOptions, prepare, simulate_prepared
from .generators import SortInstance, SubsetSumInstance, gen_random, gen_sort, gen_subset_sum
from .matrices import storage_bytes, storage_elements
from .model import SNPSystem
from .selection import SeededRandom

CSV_HEADER = "model,family,size,format,steps,wall_ms,elements,bytes,halt,seed,rep"

FAMILIES = ("sort", "subsetsum", "random")


@dataclass(frozen=True)
class BenchRecord:
    """One CSV row (bench.py:29-51)."""

    model: str
    family: str
    size: int
    format: str
    steps: int
    wall_ms: float
    elements: int
    bytes: int
    halt: str
    seed: int
    rep: int

    def csv_row(self) -> str:
        return ",".join([self.model, self.family, str(self.size), self.format, str(self.steps),
                         f"{self.wall_ms:.3f}", str(self.elements), str(self.bytes), self.halt,
                         str(self.seed), str(self.rep)])


def build_family_system(family: str, size: int, seed: int) -> SNPSystem:
    """One family member; ``size`` is n, or the neuron bound for ``random``
    (bench.py:54-64)."""
    builders = {
        "sort": lambda: gen_sort(SortInstance(size)),
        "subsetsum": lambda: gen_subset_sum(SubsetSumInstance.random(size, seed)),
        "random": lambda: gen_random(size, 4, 8, 20, 3, seed),
    }
    if family not in builders:
        raise ValueError(f"unknown family {family!r}")
    return builders[family]()


def run_bench(family: str, sizes: list[int], formats: list[Format], repetitions: int, max_steps: int,
              seed: int = 0, workers: int = 1, log=None, variant: str = "auto") -> list[BenchRecord]:
    """Time every (size, format, repetition) cell (bench.py:67-101).
    SeededRandom(seed) selection; ``log`` gets one line per cell."""
    if repetitions < 1:
        raise ValueError(f"repetitions must be >= 1, got {repetitions}")
    out: list[BenchRecord] = []
    for size in sizes:
        system = build_family_system(family, size, seed)
        name = f"{family}-{size}"
        for fmt in formats:
            t0 = time.perf_counter()
            prep = prepare(system, fmt, variant=variant if fmt is Format.COMPRESSED else "auto")
            build_ms = (time.perf_counter() - t0) * 1e3
            elements, nbytes = storage_elements(fmt, system), storage_bytes(fmt, system)
            options = SimOptions(max_steps=max_steps, selection=SeededRandom(seed), workers=workers)
            for rep in range(1, repetitions + 1):
                t0 = time.perf_counter()
                trace = simulate_prepared(prep, options)
                wall_ms = (time.perf_counter() - t0) * 1e3
                out.append(BenchRecord(name, family, size, fmt.value, trace.steps, wall_ms, elements, nbytes,
                                       trace.halt_reason.value, seed, rep))
            if log is not None:
                log(f"{name} {fmt.value}: build_ms={build_ms:.3f} elements={elements} "
                    f"last_wall_ms={out[-1].wall_ms:.3f}")
    return out


def records_to_csv(records: list[BenchRecord]) -> str:
    return "\n".join([CSV_HEADER, *(r.csv_row() for r in records)]) + "\n"
