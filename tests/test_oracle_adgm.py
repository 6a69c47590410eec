"""Pins for the ADG-M oracle (oracle/oracle.c orc_adg_m; NEXT-3 of SURVEY.md §8(f)):
hand-derived worked examples, the closed-form round count, the ADG-M
certificate (from round[] alone), Lemma "ADG-M is a partial 4-approximate
degeneracy ordering" and its Corollary K <= 4d + 1."""
import json
import os

import numpy as np
import pytest

import graphgen as gg
import oracle as O
from _refcheck import (adg_m_certificate, all_graphs, approx4_ok, degeneracy_bruteforce, is_proper,
                       jp_certificate)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_hand_examples():
    for c in json.load(open(os.path.join(GOLDEN, "adg_m_examples.json")))["cases"]:
        g = gg.from_edges(c["n"], c["edges"])
        rnd, st = O.adg_m(g)
        assert rnd.tolist() == c["rounds"], c["id"]
        assert st["T"] == c["T"], c["id"]
        assert adg_m_certificate(g, rnd) is None, c["id"]


def test_round_count_closed_form():
    # |R_l| = ceil(|U_l|/2) => |U_{l+1}| = floor(|U_l|/2) => T = floor(log2 n) + 1
    for n in list(range(0, 40)) + [1000, 1023, 1024, 1025, 4097]:
        g = gg.er(n, min(3 * n, n * (n - 1) // 2), 7) if n > 1 else gg.from_edges(n, [])
        rnd, st = O.adg_m(g)
        assert st["T"] == (n.bit_length() if n else 0), n
        sizes = np.bincount(rnd, minlength=st["T"] + 1)[1:] if n else np.zeros(0)
        u = n
        for l in range(st["T"]):
            assert sizes[l] == (u + 1) // 2
            u -= sizes[l]
        assert st["sum_active"] == sum(n >> i for i in range(st["T"]))   # |U_l| = floor(n / 2^(l-1))


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_exhaustive_small_graphs(n):
    for edges in all_graphs(n):
        g = gg.from_edges(n, edges)
        rnd, st = O.adg_m(g)
        assert adg_m_certificate(g, rnd) is None
        d = degeneracy_bruteforce(g)
        assert approx4_ok(g, rnd, d)
        for seed in (1, 2):
            color, K = O.jp(g, rnd, seed)
            assert jp_certificate(g, rnd, color, seed) is None
            assert K <= 4 * d + 1


@pytest.mark.parametrize("kind", ["er", "rmat", "grid"])
def test_random_graphs(kind):
    for seed in range(1, 4):
        g = {"er": lambda: gg.er(3000, 15000, seed), "rmat": lambda: gg.rmat(11, 8, seed=seed),
             "grid": lambda: gg.grid(48, seed=seed)}[kind]()
        rnd, st = O.adg_m(g)
        assert adg_m_certificate(g, rnd) is None
        assert st["T"] == g.n.bit_length()
        d = O.degeneracy(g)
        assert approx4_ok(g, rnd, d)
        color, K = O.jp(g, rnd, seed)
        assert is_proper(g, color) and K <= 4 * d + 1
