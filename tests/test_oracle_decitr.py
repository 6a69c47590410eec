"""Pins for the DEC-ADG-ITR oracle (oracle/oracle.c orc_dec_adg_itr; NEXT-2 of
SURVEY.md §8(f); PAPER.md:1957-1972 with SIM-COL, 1453-1477; readings Q23-Q24):
hand-derived runs, the clique closed form, equality with JP-ADG when every ADG
partition is an independent set, properness and the paper's (2(1+eps)d + 1)
color bound, the pass bound, and an independent re-implementation on small
graphs."""
import numpy as np
import pytest

import graphgen as gg
import oracle as O
from _refcheck import MASK64, all_graphs, color_bound, degeneracy_bruteforce, is_proper, splitmix64_py


def h(seed, v):
    return splitmix64_py((seed ^ v) & MASK64)


def dec_itr_py(g, rnd, seed):
    """SIM-COL-ITR partition by partition, written from the listings with sets."""
    adj = [set(g.col[g.off[v]:g.off[v + 1]].tolist()) for v in range(g.n)]
    color = {}
    for l in range(int(max(rnd)) if g.n else 0, 0, -1):
        U = {v for v in range(g.n) if rnd[v] == l}
        B = {v: {color[u] for u in adj[v] if u in color} for v in U}
        while U:
            C = {}
            for v in U:
                c = 1
                while c in B[v]:
                    c += 1
                C[v] = c
            fixed = {v for v in U if not any(u in U and C[u] == C[v] and h(seed, u) > h(seed, v)
                                             for u in adj[v])}
            for v in fixed:
                color[v] = C[v]
            for v in U - fixed:
                B[v] |= {C[u] for u in adj[v] if u in fixed}
            U -= fixed
    return [color[v] for v in range(g.n)]


def test_hand_examples():
    # K2, one partition: both pick 1, the higher hash keeps it, the other takes 2 next pass
    g = gg.from_edges(2, [(0, 1)])
    for seed in (1, 2, 3):
        rnd, _ = O.adg(g, 1, 10)
        color, K, passes = O.dec_adg_itr(g, rnd, seed)
        want = [1, 2] if h(seed, 0) > h(seed, 1) else [2, 1]
        assert color.tolist() == want and K == 2 and passes == 2
    # star: the center is its own (last) partition -> 1; leaves 2 in one pass
    g = gg.from_edges(5, [(0, i) for i in range(1, 5)])
    rnd, _ = O.adg(g, 1, 10)
    color, K, passes = O.dec_adg_itr(g, rnd, 7)
    assert color.tolist() == [1, 2, 2, 2, 2] and passes == 2


def test_clique_is_hash_rank():
    n = 9
    g = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    for seed in (1, 5):
        rnd, _ = O.adg(g, 1, 10)
        color, K, passes = O.dec_adg_itr(g, rnd, seed)
        assert color.tolist() == [1 + sum(h(seed, u) > h(seed, v) for u in range(n)) for v in range(n)]
        assert passes == n


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_exhaustive_small_graphs(n):
    for edges in all_graphs(n):
        g = gg.from_edges(n, edges)
        d = degeneracy_bruteforce(g)
        for num, den in [(1, 10), (1, 2)]:
            rnd, st = O.adg(g, num, den)
            for seed in (1, 2):
                color, K, passes = O.dec_adg_itr(g, rnd, seed)
                assert color.tolist() == dec_itr_py(g, rnd, seed)
                assert is_proper(g, color) and K <= color_bound(num, den, d)
                assert passes <= n
                src = np.repeat(np.arange(n), np.diff(g.off))
                if not (rnd[src] == rnd[g.col]).any():   # every partition independent
                    assert np.array_equal(color, O.jp(g, rnd, seed)[0])


@pytest.mark.parametrize("kind", ["er", "rmat", "grid"])
def test_random_graphs(kind):
    for seed in range(1, 4):
        g = {"er": lambda: gg.er(1500, 9000, seed), "rmat": lambda: gg.rmat(10, 8, seed=seed),
             "grid": lambda: gg.grid(30, seed=seed)}[kind]()
        d = O.degeneracy(g)
        for num, den in [(1, 100), (1, 10), (1, 2)]:
            rnd, _ = O.adg(g, num, den)
            color, K, passes = O.dec_adg_itr(g, rnd, seed)
            assert is_proper(g, color) and K <= color_bound(num, den, d) and K <= int(g.degrees().max()) + 1
            if g.n <= 1500:
                assert color.tolist() == dec_itr_py(g, rnd, seed)
