"""Pins for the CPU oracle (oracle/oracle.c) against what the paper and the
mathematics fix -- never against the oracle itself.

  * published SplitMix64 output vectors (the tie-break hash)
  * Appendix B hand-derived worked examples of Alg. 1 / Alg. 3 (tests/golden)
  * the ADG certificate (Alg. 1 as a closed-form characterisation)
  * the JP certificate (Alg. 3 GetColor fixed point) and an independent greedy
  * Lemma 1 exact round bound + per-round shrink, Lemma 4, Corollary 1, Delta+1
  * exact degeneracy vs. brute force over all induced subgraphs; chi vs. brute force
  * relabelling invariance of ADG rounds
  * exhaustive enumeration of every labelled graph on <= 6 vertices
"""
import json
import os

import numpy as np
import pytest

import graphgen as gg
import oracle as O
from _refcheck import (MASK64, adg_certificate, all_graphs, approx_ratio_ok, chromatic_bruteforce,
                       color_bound, degeneracy_bruteforce, greedy_in_order, is_proper,
                       jp_certificate, jp_certificate_np, round_bound_T0, splitmix64_py)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
GAMMA = 0x9E3779B97F4A7C15
EPS_SET = [(1, 100), (1, 10), (1, 2), (1, 1), (4294967295, 1)]


def h(seed, v):
    return splitmix64_py((seed ^ v) & MASK64)


# ------------------------------------------------------------ splitmix64 ----
def test_splitmix64_published_vectors():
    d = json.load(open(os.path.join(GOLDEN, "splitmix64_vectors.json")))
    for seq in d["sequences"]:
        for k, out in enumerate(seq["outputs"]):
            state = (seq["state"] + k * GAMMA) & MASK64
            assert O.splitmix64(state) == int(out, 0)
            assert splitmix64_py(state) == int(out, 0)


def test_splitmix64_injective_on_consecutive_ids():
    # every step of SplitMix64 is a bijection on 2^64, so no two ids collide:
    # ties in rho_R are impossible.  Spot-check 2^20 ids.
    from _refcheck import _hash_np
    hs = _hash_np(1 << 20, 1)
    assert len(np.unique(hs)) == 1 << 20
    for v in (0, 1, 12345, (1 << 20) - 1):
        assert int(hs[v]) == O.splitmix64(1 ^ v)


# ------------------------------------------------------------ Appendix B ----
def _color_rule_ok(rule, n, edges, color, seed):
    if rule == "p3_flat":
        hs = [h(seed, v) for v in range(3)]
        want = [2, 1, 2] if hs[1] == max(hs) else [1, 2, 1]
        return list(color) == want
    if rule == "p4":
        want = [2, 1, 2, 1] if h(seed, 1) > h(seed, 2) else [1, 2, 1, 2]
        return list(color) == want
    if rule == "clique_rank":
        hs = [h(seed, v) for v in range(n)]
        return all(color[v] == 1 + sum(1 for u in range(n) if hs[u] > hs[v]) for v in range(n))
    if rule == "proper_only":
        return len(set(int(c) for c in color)) == 3
    if rule == "k4_pendant_10":
        order = sorted([1, 2, 3], key=lambda v: -h(seed, v))
        return color[0] == 1 and color[4] == 2 and [color[v] for v in order] == [2, 3, 4]
    if rule == "k4_pendant_100":
        order = sorted(range(4), key=lambda v: -h(seed, v))
        ok = [color[v] for v in order] == [1, 2, 3, 4]
        return ok and color[4] == (2 if color[0] == 1 else 1)
    if rule == "k4_isolated":
        order = sorted(range(4), key=lambda v: -h(seed, v))
        return [color[v] for v in order] == [1, 2, 3, 4] and color[4] == 1
    if rule == "c10_isolated":
        return color[10] == 1 and max(color[:10]) in (2, 3)
    if rule == "jp_r":
        g = gg.from_edges(n, edges)
        order = sorted(range(n), key=lambda v: -h(seed, v))
        return list(color) == greedy_in_order(g, order)
    raise KeyError(rule)


@pytest.mark.parametrize("seed", [1, 2, 7, 0xDEADBEEFCAFEF00D])
def test_appendix_b(seed):
    cases = json.load(open(os.path.join(GOLDEN, "appendix_b.json")))["cases"]
    for c in cases:
        g = gg.from_edges(c["n"], c["edges"])
        num, den = c["eps"]
        rnd, st = O.adg(g, num, den)
        assert rnd.tolist() == c["rounds"], c["id"]
        assert st["T"] == c["T"], c["id"]
        color, K = O.jp(g, rnd, seed)
        if "colors" in c:
            assert color.tolist() == c["colors"], c["id"]
        if "color_rule" in c:
            assert _color_rule_ok(c["color_rule"], c["n"], c["edges"], color.tolist(), seed), c["id"]
        if "K" in c:
            assert K == c["K"], c["id"]
        assert K == (int(color.max()) if c["n"] else 0)


def test_appendix_b_per_round_trace():
    # B11: (|U|, S, |R|) per round = (5, 14, 1), (4, 12, 4)
    g = gg.from_edges(5, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (4, 0)])
    _, st = O.adg(g, 1, 100, per_round=True)
    assert st["nU"].tolist() == [5, 4] and st["S"].tolist() == [14, 12] and st["nR"].tolist() == [1, 4]


def test_threshold_is_le_not_lt():
    # B13: equality den*D*n == (den+num)*S must select; '<' gives T=2
    g = gg.from_edges(11, [(i, (i + 1) % 10) for i in range(10)])
    rnd, st = O.adg(g, 1, 10)
    assert st["T"] == 1 and (rnd == 1).all()


# ------------------------------------------------------------ certificates --
def _full_check(g, num, den, seed, d=None, chi=None):
    rnd, st = O.adg(g, num, den, per_round=True)
    T = st["T"]
    assert adg_certificate(g, rnd, num, den) is None
    # Lemma 1: exact integer round bound and per-round shrink
    assert T <= round_bound_T0(g.n, num, den)
    nU = st["nU"].tolist() + [0]
    for l in range(T):
        assert nU[l + 1] * (den + num) < nU[l] * den or nU[l + 1] == 0
        assert st["nR"][l] >= 1
    # Lemma 2: sum |U_l| <= (1+eps)/eps * n
    assert st["sum_active"] * num <= (den + num) * g.n
    color, K = O.jp(g, rnd, seed)
    assert (jp_certificate(g, rnd, color, seed) if g.n <= 64 else
            jp_certificate_np(g, rnd, color, seed)) is None
    assert is_proper(g, color)
    deg = g.degrees()
    Delta = int(deg.max()) if g.n else 0
    assert K <= Delta + 1
    if d is None:
        d = O.degeneracy(g)
    assert approx_ratio_ok(g, rnd, num, den, d)        # Lemma 4
    assert K <= color_bound(num, den, d)              # Corollary 1
    if chi is not None:
        assert K >= chi
    return rnd, color, T, K


@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 5])
def test_exhaustive_small_graphs(n):
    for edges in all_graphs(n):
        g = gg.from_edges(n, edges)
        d = degeneracy_bruteforce(g)
        assert O.degeneracy(g) == d
        chi = chromatic_bruteforce(g)
        assert O.brute_chi(g) == chi
        for num, den in EPS_SET:
            for seed in (1, 2):
                rnd, color, T, K = _full_check(g, num, den, seed, d=d, chi=chi)
                if num == 4294967295:       # eps -> infinity: JP-ADG = JP-R
                    assert T == min(n, 1)
                    order = sorted(range(n), key=lambda v: -h(seed, v))
                    assert color.tolist() == greedy_in_order(g, order)


def test_exhaustive_n6():
    n = 6
    for edges in all_graphs(n):
        g = gg.from_edges(n, edges)
        num, den = (1, 10)
        rnd, st = O.adg(g, num, den)
        assert adg_certificate(g, rnd, num, den) is None
        color, K = O.jp(g, rnd, 3)
        assert jp_certificate(g, rnd, color, 3) is None
        assert K >= O.brute_chi(g)


@pytest.mark.parametrize("seed", range(10))
def test_random_small_with_brute_chi(seed):
    rng = np.random.default_rng(seed)
    for n in (7, 9, 12):
        p = rng.uniform(0.1, 0.8)
        edges = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        g = gg.from_edges(n, edges)
        d = O.degeneracy(g)
        if n <= 9:
            assert d == degeneracy_bruteforce(g)
        chi = O.brute_chi(g)
        for num, den in EPS_SET:
            _full_check(g, num, den, seed + 1, d=d, chi=chi)


@pytest.mark.parametrize("kind", ["er", "rmat"])
def test_random_medium(kind):
    for seed in range(1, 6):
        g = gg.er(2000, 12000, seed) if kind == "er" else gg.rmat(11, 8, seed=seed)
        for num, den in [(1, 100), (1, 10), (1, 2)]:
            _full_check(g, num, den, seed)


def test_config1_er_certificates():
    g = gg.config_graph("er")
    _full_check(g, 1, 10, 1)


# ------------------------------------------------------------ degeneracy ----
def test_degeneracy_textbook_values():
    def clique(n):
        return gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    assert O.degeneracy(clique(7)) == 6
    assert O.degeneracy(gg.from_edges(9, [(i, (i + 1) % 9) for i in range(9)])) == 2
    assert O.degeneracy(gg.from_edges(6, [(0, i) for i in range(1, 6)])) == 1
    W = 20
    grid = [(i * W + j, i * W + j + 1) for i in range(W) for j in range(W - 1)] + \
           [(i * W + j, (i + 1) * W + j) for i in range(W - 1) for j in range(W)]
    assert O.degeneracy(gg.from_edges(W * W, grid)) == 2
    petersen = [(i, (i + 1) % 5) for i in range(5)] + [(5 + i, 5 + (i + 2) % 5) for i in range(5)] + \
               [(i, i + 5) for i in range(5)]
    P = gg.from_edges(10, petersen)
    assert O.degeneracy(P) == 3 and O.brute_chi(P) == 3
    assert O.brute_chi(clique(4)) == 4
    assert O.brute_chi(gg.from_edges(5, [(i, (i + 1) % 5) for i in range(5)])) == 3


def test_degeneracy_bounds_on_generated():
    # d <= Delta and 4m >= d^2
    for g in (gg.er(3000, 20000, 3), gg.rmat(12, 8, seed=3), gg.grid(64, seed=3)):
        d = O.degeneracy(g)
        assert d <= int(g.degrees().max())
        assert 4 * g.m >= d * d


# ------------------------------------------------------------ invariances ---
def test_adg_rounds_invariant_under_relabelling():
    g = gg.rmat(11, 8, seed=5)
    perm = np.random.default_rng(0).permutation(g.n)
    src = np.repeat(np.arange(g.n), np.diff(g.off))
    edges = np.stack([perm[src], perm[g.col]], axis=1)
    g2 = gg.from_edges(g.n, edges)
    for num, den in [(1, 100), (1, 10), (1, 2)]:
        r1, _ = O.adg(g, num, den)
        r2, _ = O.adg(g2, num, den)
        assert (r2[perm] == r1).all()


def test_clique_colors_are_hash_ranks():
    n = 12
    g = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    for seed in (1, 99):
        rnd, _ = O.adg(g, 1, 10)
        color, K = O.jp(g, rnd, seed)
        hs = [h(seed, v) for v in range(n)]
        assert color.tolist() == [1 + sum(1 for u in range(n) if hs[u] > hs[v]) for v in range(n)]
        assert K == n


def test_jp_arbitrary_first_key():
    # pgc_jp_color accepts any int32 first key: constant key = JP-R, degree key = JP-LF
    g = gg.er(300, 1500, 4)
    seed = 5
    const = np.zeros(g.n, dtype=np.int32)
    color, _ = O.jp(g, const, seed)
    order = sorted(range(g.n), key=lambda v: -h(seed, v))
    assert color.tolist() == greedy_in_order(g, order)
    deg = g.degrees().astype(np.int32)
    color, _ = O.jp(g, deg, seed)
    order = sorted(range(g.n), key=lambda v: (-int(deg[v]), -h(seed, v)))
    assert color.tolist() == greedy_in_order(g, order)


def test_jp_levels_longest_path():
    # level[v] = 1 + max level over preds: J for a clique of n is n; a star is 2
    n = 9
    g = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    rnd = np.ones(n, dtype=np.int32)
    _, _, lvl, J = O.jp(g, rnd, 1, levels=True)
    assert J == n and sorted(lvl.tolist()) == list(range(1, n + 1))
    g = gg.from_edges(6, [(0, i) for i in range(1, 6)])
    rnd, _ = O.adg(g, 1, 10)
    _, _, lvl, J = O.jp(g, rnd, 1, levels=True)
    assert J == 2 and lvl[0] == 1


@pytest.mark.parametrize("n", [2, 3, 7, 600, 1001])
def test_path_peels_two_ends_per_round(n):
    """Closed form (Alg. 1): on the path P_n with eps < 1/(n-1),
    a sub-path of n' >= 3 vertices has mean degree 2(n'-1)/n' and
    (1+eps) * 2(n'-1)/n' < 2, so only its two ends (degree 1) leave in a round;
    hence round[i] = min(i, n-1-i) + 1 and T = ceil(n/2).  n = 600, 1001 give
    more than 255 rounds (the GPU's one-byte round state wraps there)."""
    g = gg.from_edges(n, [(i, i + 1) for i in range(n - 1)])
    r, st = O.adg(g, 1, 10 * n)
    i = np.arange(n)
    assert st["T"] == (n + 1) // 2
    assert np.array_equal(r, np.minimum(i, n - 1 - i) + 1)
    # every edge joins two rounds except the middle one of an even path
    assert st["cross_edges"] == (n - 1) - (1 if n % 2 == 0 else 0)
