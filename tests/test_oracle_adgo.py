"""Pins for the ADG-O oracle (oracle/oracle.c orc_adg_o, orc_jp_rho; NEXT-1 of
SURVEY.md §8(f)): hand-derived runs of the ADG-O listing, rounds equal to
ADG's (same PARTITION rule), rho = the (round, D_rem, id) removal order from
round[] alone, rank = number of higher-rho neighbours, the JP fixed point for
rho, Corollary 1's bound (any tie-break inside ADG's rounds) and brute chi."""
import json
import os

import numpy as np
import pytest

import graphgen as gg
import oracle as O
from _refcheck import (adg_o_rho_check, all_graphs, chromatic_bruteforce, color_bound,
                       degeneracy_bruteforce, is_proper, jp_certificate_rho)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
EPS = [(1, 100), (1, 10), (1, 2)]


def test_hand_examples():
    for c in json.load(open(os.path.join(GOLDEN, "adg_o_examples.json")))["cases"]:
        g = gg.from_edges(c["n"], c["edges"])
        rnd, rho, rank, drem, T = O.adg_o(g, *c["eps"])
        assert rnd.tolist() == c["rounds"] and rho.tolist() == c["rho"], c["id"]
        assert rank.tolist() == c["rank"], c["id"]
        color, K = O.jp_rho(g, rho)
        assert color.tolist() == c["colors"] and K == c["K"], c["id"]


def _check(g, num, den, d=None, chi=None):
    rnd, rho, rank, drem, T = O.adg_o(g, num, den)
    r_adg, st = O.adg(g, num, den)
    assert np.array_equal(rnd, r_adg) and T == st["T"]
    assert adg_o_rho_check(g, rnd, rho) is None
    src = np.repeat(np.arange(g.n), np.diff(g.off))
    up = np.bincount(src[rho[g.col] > rho[src]], minlength=g.n)
    assert np.array_equal(rank, up)                        # UPDATEandPRIORITIZE's rank
    color, K = O.jp_rho(g, rho)
    if g.n <= 3000:
        assert jp_certificate_rho(g, rho, color) is None
    assert is_proper(g, color)
    if d is None:
        d = O.degeneracy(g)
    assert K <= color_bound(num, den, d)
    if chi is not None:
        assert K >= chi
    return K


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_exhaustive_small_graphs(n):
    for edges in all_graphs(n):
        g = gg.from_edges(n, edges)
        d, chi = degeneracy_bruteforce(g), chromatic_bruteforce(g)
        for num, den in EPS:
            _check(g, num, den, d, chi)


@pytest.mark.parametrize("kind", ["er", "rmat", "grid"])
def test_random_graphs(kind):
    for seed in range(1, 4):
        g = {"er": lambda: gg.er(2500, 12000, seed), "rmat": lambda: gg.rmat(11, 8, seed=seed),
             "grid": lambda: gg.grid(40, seed=seed)}[kind]()
        for num, den in EPS:
            _check(g, num, den)
