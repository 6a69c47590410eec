"""Pins for the JP baseline orderings (NEXT-4 of SURVEY.md
§8(f)): JP with the first keys of JP-FF / JP-LF / JP-LLF / JP-R equals the
textbook sequential greedy in that priority order, computed
here independently of the oracle."""
import math

import numpy as np
import pytest

import graphgen as gg
import oracle as O
from _refcheck import MASK64, greedy_in_order, is_proper, splitmix64_py


def baseline_key(g, kind):
    deg = g.degrees()
    if kind == "ff":
        return -np.arange(g.n, dtype=np.int64)
    if kind == "lf":
        return deg.astype(np.int64)
    if kind == "llf":
        return np.array([math.ceil(math.log2(d)) if d > 1 else 0 for d in deg], dtype=np.int64)
    return np.zeros(g.n, dtype=np.int64)


@pytest.mark.parametrize("kind", ["r", "ff", "lf", "llf"])
def test_baselines_are_greedy_in_priority_order(kind):
    for seed, g in [(1, gg.er(400, 2400, 3)), (5, gg.rmat(9, 8, seed=4)), (9, gg.grid(20, seed=2))]:
        key = baseline_key(g, kind)
        color, K = O.jp(g, key.astype(np.int32), seed)
        order = sorted(range(g.n), key=lambda v: (-int(key[v]), -splitmix64_py((seed ^ v) & MASK64)))
        assert color.tolist() == greedy_in_order(g, order)
        assert is_proper(g, color) and K <= int(g.degrees().max()) + 1


def test_ff_is_the_natural_order_greedy():
    # JP-FF needs no hash: the path 0-1-2-...-9 alternates 1, 2; K_n is 1..n in id order
    g = gg.from_edges(10, [(i, i + 1) for i in range(9)])
    color, K = O.jp(g, baseline_key(g, "ff").astype(np.int32), 123)
    assert color.tolist() == [1, 2] * 5 and K == 2
    n = 7
    g = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    color, _ = O.jp(g, baseline_key(g, "ff").astype(np.int32), 5)
    assert color.tolist() == list(range(1, n + 1))
