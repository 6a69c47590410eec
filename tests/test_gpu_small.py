"""GPU parity of the one-kernel small-graph path (csrc/small.cu): JP-ADG as ONE
persistent cooperative kernel -- ADG rounds (Alg. 1) and
frontier-driven JP levels with count[] decrements (Alg. 3)
separated by grid barriers -- against the CPU oracle, bit-exact (round[],
color[], T, K, sum |U_l|, X, sum |pred|, J).

The path is forced on for every graph here (the default heuristic picks it
for small low-degree graphs only); test_gpu_parity.py covers the
multi-kernel path with it forced off.
"""
import json
import os

import numpy as np
import pytest
import torch

import graphgen as gg
import oracle as O
from _refcheck import all_graphs

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


VARIANT = {"v": None}


@pytest.fixture(autouse=True, params=["grid", "cluster", "cluster-levels"])
def small_path(request):
    """Both variants of the path: the cooperative grid kernel (k_small_jp_adg)
    and the one-cluster kernel with the state in distributed shared memory
    (k_tiny_jp_adg, taken whenever the graph fits the cluster)."""
    pgc = pytest.importorskip("paper_2008_11321_b200")
    pgc.set_tuning("small_max_arcs", 1 << 40)
    pgc.set_tuning("small_max_avg", 1 << 30)
    if request.param == "grid":
        pgc.set_tuning("tiny_max_n", 0)
    else:
        pgc.set_tuning("tiny_max_n", 1 << 30)
        pgc.set_tuning("tiny_max_arcs", 1 << 40)
        # the cluster kernel's JP: barrier-free dataflow (default) or frontier levels
        pgc.set_tuning("tiny_dataflow", 0 if request.param == "cluster-levels" else 1)
    VARIANT["v"] = request.param
    yield pgc
    pgc.set_tuning("small_max_arcs", 1 << 24)
    pgc.set_tuning("small_max_avg", 20)
    pgc.set_tuning("small_blocks_per_sm", 0)
    pgc.set_tuning("tiny_max_n", 1 << 17)
    pgc.set_tuning("tiny_max_arcs", 1 << 22)
    pgc.set_tuning("tiny_dataflow", 1)
    pgc.set_tuning("levels", 0)


def dev(g):
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda() if g.nnz else torch.empty(0, dtype=torch.int32, device="cuda")
    return off, col


def assert_parity(pgc, g, num, den, seed, levels=True):
    off, col = dev(g)
    pgc.set_tuning("levels", 1 if levels else 0)
    rnd, color, T, K = pgc.color_jp_adg(off, col, num, den, seed)
    torch.cuda.synchronize()
    st = pgc.last_stats()
    if g.n == 0:
        assert st["small_path"] == 0
    elif VARIANT["v"] == "grid":
        assert st["small_path"] == 1
    elif g.n <= 20000 and g.nnz <= 300000:   # fits 16 CTAs' shared memory (arrays + own rows)
        assert st["small_path"] == 2 and st["core_ctas"] >= 2
    else:   # the cluster kernel when it fits, else the grid kernel
        assert st["small_path"] in (1, 2)
    r_or, st_or = O.adg(g, num, den)
    c_or, K_or, _, J_or = O.jp(g, r_or, seed, levels=True)
    r_gpu, c_gpu = rnd.cpu().numpy(), color.cpu().numpy()
    assert T == st_or["T"]
    bad = np.nonzero(r_gpu != r_or)[0]
    assert len(bad) == 0, f"round mismatch at {bad[:10]} gpu={r_gpu[bad[:10]]} cpu={r_or[bad[:10]]}"
    bad = np.nonzero(c_gpu != c_or)[0]
    assert len(bad) == 0, f"color mismatch at {bad[:10]} gpu={c_gpu[bad[:10]]} cpu={c_or[bad[:10]]}"
    assert K == K_or
    assert st["rounds"] == T and st["num_colors"] == K
    assert st["sum_active"] == st_or["sum_active"]
    assert st["cross_edges"] == st_or["cross_edges"]
    assert st["pred_arcs"] == g.m
    if levels:
        assert st["jp_levels"] == J_or, (st["jp_levels"], J_or)
    if g.n > 0:
        assert st["kernel_launches"] == 1
    return T, K


def test_appendix_b_cases(small_path):
    cases = json.load(open(os.path.join(GOLDEN, "appendix_b.json")))["cases"]
    for c in cases:
        g = gg.from_edges(c["n"], c["edges"])
        for seed in (1, 2, 0xDEADBEEFCAFEF00D):
            T, K = assert_parity(small_path, g, c["eps"][0], c["eps"][1], seed)
            assert T == c["T"]


def test_zoo_all_graphs_up_to_5(small_path):
    edges, n = [], 0
    for k in range(1, 6):
        for es in all_graphs(k):
            edges += [(a + n, b + n) for a, b in es]
            n += k
    g = gg.from_edges(n, edges)
    for num, den in [(1, 100), (1, 10), (1, 2), (1, 1), (4294967295, 1)]:
        assert_parity(small_path, g, num, den, 7)


@pytest.mark.parametrize("seed", range(1, 7))
def test_random_er_rmat(small_path, seed):
    for g in (gg.er(3000, 15000 + 1000 * seed, seed), gg.rmat(8 + seed % 7, 8, seed=seed)):
        for num, den in [(1, 100), (1, 10), (1, 2)]:
            assert_parity(small_path, g, num, den, seed * 31 + 1)


def test_cliques_hubs_and_windows(small_path):
    # K_n: colors up to n -> several 64-color windows per vertex; J = n
    for n in (70, 300, 700):
        g = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
        T, K = assert_parity(small_path, g, 1, 10, 3)
        assert T == 1 and K == n
    # star (one warp owner with 5000 arcs) and a hub joined to a clique
    assert_parity(small_path, gg.from_edges(5001, [(0, i) for i in range(1, 5001)]), 1, 10, 3)
    n = 400
    edges = [(i, j) for i in range(1, n) for j in range(i + 1, n)] + [(0, i) for i in range(1, 20000)]
    assert_parity(small_path, gg.from_edges(20000, edges), 1, 100, 5)


def test_edge_cases(small_path):
    off, col = dev(gg.from_edges(0, []))
    r, c, T, K = small_path.color_jp_adg(off, col, 1, 10, 1)
    assert T == 0 and K == 0 and r.numel() == 0
    for n in (1, 2, 33, 1000, 70000):   # edgeless: one round, every color 1, J = 1
        assert_parity(small_path, gg.from_edges(n, []), 1, 10, 1)
    # a single edge among many isolated vertices, and ragged warp tails
    for n in (2, 31, 32, 33, 513, 1025):
        assert_parity(small_path, gg.from_edges(n, [(0, n - 1)]), 1, 10, 2)


def test_more_than_255_rounds(small_path):
    for n in (1000, 1001):
        edges = [(i, i + 1) for i in range(n - 1)] + [(n + i, n + i + 1) for i in range(600)]
        perm = np.random.default_rng(n).permutation(n + 601)
        g = gg.from_edges(n + 601, [(int(perm[a]), int(perm[b])) for a, b in edges])
        T, _ = assert_parity(small_path, g, 1, 100 * n, 3)
        assert T > 255


@pytest.mark.parametrize("bps", [1, 2])
def test_grid_sizes(small_path, bps):
    # results never depend on the grid (1 block per SM forces several vertices per warp)
    small_path.set_tuning("small_blocks_per_sm", bps)
    assert_parity(small_path, gg.rmat(12, 16, seed=5), 1, 10, 9)
    assert_parity(small_path, gg.er(50000, 400000, 4), 1, 2, 9)


@pytest.mark.parametrize("name", ["er", "grid", "rmat20"])
def test_config_parity(small_path, name):
    g = gg.config_graph(name)
    for num, den in gg.CONFIGS[name][1]:
        assert_parity(small_path, g, num, den, 1)


def test_default_heuristic_and_host_api(small_path):
    """Defaults: ER takes the one-cluster kernel, the grid the cooperative grid
    kernel, R-MAT 20 (mean degree 30, a deep dense core) the multi-kernel
    path; the host-buffer entry point gives the same result on the small path."""
    if VARIANT["v"] != "grid":
        pytest.skip("defaults: checked once")
    pgc = small_path
    for k, v in (("small_max_arcs", 1 << 24), ("small_max_avg", 20), ("tiny_max_n", 1 << 17),
                 ("tiny_max_arcs", 1 << 22)):
        pgc.set_tuning(k, v)
    for name, want in (("er", 2), ("grid", 1), ("rmat20", 0)):
        g = gg.config_graph(name)
        off, col = dev(g)
        num, den = gg.CONFIGS[name][1][0]
        rnd, color, T, K = pgc.color_jp_adg(off, col, num, den, 1)
        torch.cuda.synchronize()
        assert pgc.last_stats()["small_path"] == want, name
        if name == "er":
            h_r = torch.zeros(g.n, dtype=torch.int32).pin_memory()
            h_c = torch.zeros(g.n, dtype=torch.int32).pin_memory()
            T2, K2 = pgc.color_jp_adg_host(torch.from_numpy(g.off), torch.from_numpy(g.col), num, den,
                                           1, h_r, h_c)
            assert pgc.last_stats()["small_path"] == 2
            assert (T2, K2) == (T, K)
            assert np.array_equal(h_r.numpy(), rnd.cpu().numpy())
            assert np.array_equal(h_c.numpy(), color.cpu().numpy())


def test_cluster_fallback_when_rows_do_not_fit(small_path):
    """A hub whose row does not fit its CTA's shared memory: the one-cluster
    kernel leaves (every CTA checks every peer's fit) and the grid kernel runs;
    the result is the same."""
    n = 120001
    g = gg.from_edges(n, [(0, i) for i in range(1, n)] + [(i, i + 1) for i in range(1, n - 1, 2)])
    T, K = assert_parity(small_path, g, 1, 10, 4)
    assert small_path.last_stats()["small_path"] == 1


def test_repeats_identical(small_path):
    g = gg.config_graph("er")
    off, col = dev(g)
    ref = None
    for _ in range(20):
        r, c, T, K = small_path.color_jp_adg(off, col, 1, 10, 1)
        out = (r.cpu().numpy(), c.cpu().numpy(), T, K)
        if ref is None:
            ref = out
        assert np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1]) and out[2:] == ref[2:]
