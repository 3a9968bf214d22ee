"""Native synth-v1 generator (snpio_synth_v1) against the numpy restatement
(generators.synth_v1_numpy / sharded.synth_v1_rows_numpy), which the golden
fixtures pin to the reference (tests/golden/synth.npz via make_golden.py)."""

import numpy as np
import pytest

from paper_2408_04343_b200 import generators as g
from paper_2408_04343_b200 import sharded as shd


def _same(a, b):
    for x, y in [(a.initial, b.initial), (a.adj_offsets, b.adj_offsets), (a.adj_targets, b.adj_targets),
                 (a.rule_map.offsets, b.rule_map.offsets)]:
        np.testing.assert_array_equal(x, y)
    for f in ("threshold", "is_exact", "consumed", "produced", "delay", "neuron"):
        np.testing.assert_array_equal(getattr(a.rules, f), getattr(b.rules, f))


@pytest.mark.parametrize("q,delays,seed", [(17, False, g.SYNTH_SEED), (1000, True, g.SYNTH_SEED),
                                           (65_537, True, 7), (250_000, False, 2**64 - 1)])
def test_native_equals_numpy(q, delays, seed):
    _same(g.synth_v1(q, seed, delays), g.synth_v1_numpy(q, seed, delays))


@pytest.mark.parametrize("lo,hi", [(0, 200_000), (0, 1), (1024, 77_777), (150_000, 200_000), (5, 5)])
def test_native_rows_equal_numpy(lo, hi):
    _same(shd.synth_v1_rows(200_000, lo, hi, with_delays=True),
          shd.synth_v1_rows_numpy(200_000, lo, hi, with_delays=True))


def test_too_small():
    with pytest.raises(g.InvalidInstance):
        g.synth_v1(16)
