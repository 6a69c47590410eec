"""Independent checkers used to pin the oracle (and, transitively, the CUDA path).

Nothing here calls ``oracle/`` or the CUDA library: each function restates a
closed-form characterisation from the paper in plain Python / numpy, with a
different loop structure from the peeling oracle, so that a mistake in the
oracle (a dropped term, a wrong sign or index, '<' for '<=', a reversed
priority) fails at least one of them.
"""
from __future__ import annotations

import itertools
from math import floor

import numpy as np

MASK64 = (1 << 64) - 1


def splitmix64_py(x: int) -> int:
    """SplitMix64 first output for state x; pinned by tests/golden/splitmix64_vectors.json."""
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def adjacency(g):
    off, col = g.off, g.col
    return [col[off[v]:off[v + 1]].tolist() for v in range(g.n)]


def key(rnd, seed, v):
    """JP-ADG priority <rho_ADG, rho_R>, lexicographic."""
    return (int(rnd[v]), splitmix64_py((seed ^ v) & MASK64))


# ---------------------------------------------------------------- ADG -------
def adg_certificate(g, rnd, num, den):
    """Characterisation of ADG's output (Alg. 1) from round[] alone.

    For every l = 1..T: U_l = {v : round[v] >= l}; D_l(v) = |N(v) ∩ U_l|;
    S_l = sum_{U_l} D_l; for all v in U_l:
        round[v] == l  <=>  den * D_l(v) * |U_l| <= (den + num) * S_l.
    Unique: given round[] of rounds < l, round l's set is determined.
    Returns None if valid, else a message."""
    n = g.n
    if n == 0:
        return None if len(rnd) == 0 else "n=0 but rounds given"
    rnd = np.asarray(rnd, dtype=np.int64)
    if rnd.min() < 1:
        return f"vertex {int(np.argmin(rnd))} has round < 1"
    T = int(rnd.max())
    src = np.repeat(np.arange(n), np.diff(g.off))
    dst = g.col.astype(np.int64)
    for l in range(1, T + 1):
        inU = rnd >= l
        nU = int(inU.sum())
        if nU == 0:
            return f"round {l} is empty"
        keep = inU[src] & inU[dst]
        D = np.bincount(src[keep], minlength=n)
        S = int(D[inU].sum())
        if n < 4096:   # direct product form, Python big ints
            sel = np.array([den * int(x) * nU <= (den + num) * S for x in D], dtype=bool)
        else:          # equivalent floor form for integer D >= 0
            sel = _le_exact(D, nU, S, num, den)
        want = inU & sel
        got = rnd == l
        bad = np.nonzero(want != got)[0]
        if len(bad):
            return f"round {l}: vertex {int(bad[0])} (D={int(D[bad[0]])}, |U|={nU}, S={S})"
    return None


def _le_exact(D, nU, S, num, den):
    # den*D*nU <= (den+num)*S  <=>  D <= floor((den+num)*S / (den*nU)) for integer D >= 0
    dmax = min(((den + num) * S) // (den * nU), 1 << 62)
    return D <= dmax


def round_bound_T0(n, num, den):
    """Exact integer form of Lemma 1: the smallest t with
    (den+num)^t >= n * den^t (t >= 1 when n >= 1)."""
    if n == 0:
        return 0
    t = 0
    while (den + num) ** t < n * den ** t:
        t += 1
    return max(t, 1)


# ---------------------------------------------------------------- JP --------
def jp_certificate(g, rnd, color, seed):
    """Characterisation of JP's output (Alg. 3): for every v,
    color[v] = min({1..|pred(v)|+1} minus {color[u] : u in pred(v)}) with
    pred(v) = {u in N(v) : key(u) > key(v)}.  The fixed point of this local rule
    on the DAG is unique.  Returns None if valid else a message."""
    adj = adjacency(g)
    keys = [key(rnd, seed, v) for v in range(g.n)]
    for v in range(g.n):
        preds = [u for u in adj[v] if keys[u] > keys[v]]
        used = {int(color[u]) for u in preds}
        c = 1
        while c in used:
            c += 1
        if int(color[v]) != c:
            return f"vertex {v}: color {int(color[v])} but mex of preds is {c}"
    return None


def jp_certificate_np(g, rnd, color, seed):
    """Vectorised form of jp_certificate for large graphs (numpy).  Checks that
    color[v] is absent from pred colors and that every c < color[v] occurs."""
    n = g.n
    if n == 0:
        return None
    h = np.array([splitmix64_py((seed ^ v) & MASK64) for v in range(n)], dtype=np.uint64) \
        if n <= 200000 else _hash_np(n, seed)
    rnd = np.asarray(rnd, dtype=np.int64)
    color = np.asarray(color, dtype=np.int64)
    src = np.repeat(np.arange(n), np.diff(g.off))
    dst = g.col.astype(np.int64)
    is_pred = (rnd[dst] > rnd[src]) | ((rnd[dst] == rnd[src]) & (h[dst] > h[src]))
    ps, pd = src[is_pred], dst[is_pred]
    if (color < 1).any():
        return "uncolored vertex"
    if (color[ps] == color[pd]).any():
        i = int(np.nonzero(color[ps] == color[pd])[0][0])
        return f"vertex {int(ps[i])} shares color with pred {int(pd[i])}"
    # every color below color[v] must be used by a pred: count distinct (v, c) pairs with c < color[v]
    below = color[pd] < color[ps]
    pairs = np.unique(ps[below] * (int(color.max()) + 1) + color[pd][below])
    cnt = np.bincount(pairs // (int(color.max()) + 1), minlength=n)
    bad = np.nonzero(cnt != color - 1)[0]
    if len(bad):
        return f"vertex {int(bad[0])}: color {int(color[bad[0]])} not the mex of its preds"
    return None


def _hash_np(n, seed):
    x = (np.arange(n, dtype=np.uint64) ^ np.uint64(seed & MASK64))
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def greedy_in_order(g, order):
    """Textbook sequential greedy: color vertices in the given
    order with the smallest color unused by already-colored neighbors."""
    adj = adjacency(g)
    color = [0] * g.n
    for v in order:
        used = {color[u] for u in adj[v] if color[u]}
        c = 1
        while c in used:
            c += 1
        color[v] = c
    return color


def is_proper(g, color):
    color = np.asarray(color)
    if g.n and (color < 1).any():
        return False
    src = np.repeat(np.arange(g.n), np.diff(g.off))
    return not (color[src] == color[g.col]).any()


# --------------------------------------------------------- degeneracy -------
def degeneracy_bruteforce(g):
    """d = max over nonempty vertex subsets W of min_{v in W} deg_W(v)
    (definition of d-degenerate).  n <= 12."""
    adj = [set(a) for a in adjacency(g)]
    best = 0
    for r in range(1, g.n + 1):
        for W in itertools.combinations(range(g.n), r):
            Ws = set(W)
            md = min(len(adj[v] & Ws) for v in W)
            best = max(best, md)
    return best


def chromatic_bruteforce(g):
    """chi(G) by trying all k^n assignments for increasing k (n <= 7)."""
    n = g.n
    if n == 0:
        return 0
    edges = [(v, u) for v in range(n) for u in adjacency(g)[v] if u > v]
    for k in range(1, n + 1):
        for assign in itertools.product(range(k), repeat=n):
            if all(assign[a] != assign[b] for a, b in edges):
                return k
    return n


def approx_ratio_ok(g, rnd, num, den, d):
    """Lemma 4: every v has at most 2(1+eps)d neighbors u
    with round[u] >= round[v]; exact: den*|...| <= 2*(den+num)*d."""
    src = np.repeat(np.arange(g.n), np.diff(g.off))
    dst = g.col
    rnd = np.asarray(rnd)
    later = np.bincount(src[rnd[dst] >= rnd[src]], minlength=g.n)
    return bool((den * later <= 2 * (den + num) * d).all())


def color_bound(num, den, d):
    """Corollary 1 in exact integer form: K <= floor(2(den+num)d/den) + 1."""
    return (2 * (den + num) * d) // den + 1


def all_graphs(n):
    """Every labelled simple graph on n vertices, as edge lists."""
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    for mask in range(1 << len(pairs)):
        yield [pairs[b] for b in range(len(pairs)) if mask >> b & 1]


# ---------------------------------------------------------------- ADG-M -----
def adg_m_certificate(g, rnd):
    """Characterisation of ADG-M's output (readings Q19-Q21)
    from round[] alone: for every l, with U_l = {v : round[v] >= l} and
    D_l(v) = |N(v) ∩ U_l|, round l removes exactly the ceil(|U_l|/2) vertices of
    U_l that come first in ascending (D_l, id) order.  Returns None if valid."""
    n = g.n
    if n == 0:
        return None if len(rnd) == 0 else "n=0 but rounds given"
    rnd = np.asarray(rnd, dtype=np.int64)
    if rnd.min() < 1:
        return f"vertex {int(np.argmin(rnd))} has round < 1"
    src = np.repeat(np.arange(n), np.diff(g.off))
    dst = g.col.astype(np.int64)
    for l in range(1, int(rnd.max()) + 1):
        inU = rnd >= l
        U = np.nonzero(inU)[0]
        keep = inU[src] & inU[dst]
        D = np.bincount(src[keep], minlength=n)
        first = U[np.lexsort((U, D[U]))][: (len(U) + 1) // 2]   # key (D asc, id asc)
        want = np.zeros(n, dtype=bool)
        want[first] = True
        bad = np.nonzero(want != (rnd == l))[0]
        if len(bad):
            return f"round {l}: vertex {int(bad[0])}"
    return None


def approx4_ok(g, rnd, d):
    """Lemma (ADG-M): every vertex has at most 4d neighbours
    ranked equal or higher."""
    rnd = np.asarray(rnd, dtype=np.int64)
    src = np.repeat(np.arange(g.n), np.diff(g.off))
    dst = g.col.astype(np.int64)
    up = np.bincount(src[rnd[dst] >= rnd[src]], minlength=g.n)
    return bool((up <= 4 * d).all())


# ---------------------------------------------------------------- ADG-O -----
def residual_at_removal(g, rnd):
    """D_rem(v) = |N(v) ∩ U_round(v)|: the residual degree v had when its round
    selected it (U_l = {u : round[u] >= l})."""
    rnd = np.asarray(rnd, dtype=np.int64)
    src = np.repeat(np.arange(g.n), np.diff(g.off))
    dst = g.col.astype(np.int64)
    return np.bincount(src[rnd[dst] >= rnd[src]], minlength=g.n)


def adg_o_rho_check(g, rnd, rho):
    """rho_ADG-O (reading Q22) is the removal order: rounds in
    increasing order, inside a round increasing (D_rem, id); a permutation."""
    n = g.n
    rho = np.asarray(rho, dtype=np.int64)
    if not np.array_equal(np.sort(rho), np.arange(n)):
        return "rho is not a permutation of 0..n-1"
    dr = residual_at_removal(g, rnd)
    order = np.lexsort((np.arange(n), dr, np.asarray(rnd, dtype=np.int64)))
    if not np.array_equal(rho[order], np.arange(n)):
        return "rho is not the (round, D_rem, id) order"
    return None


def jp_certificate_rho(g, rho, color):
    """Alg. 3's GetColor fixed point for a total-order priority rho (larger first)."""
    adj = adjacency(g)
    for v in range(g.n):
        used = {int(color[u]) for u in adj[v] if rho[u] > rho[v]}
        c = 1
        while c in used:
            c += 1
        if int(color[v]) != c:
            return f"vertex {v}: color {int(color[v])}, GetColor gives {c}"
    return None
