"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Everything is integer, so the bar is bit-exactness: identical round[] and
color[] per vertex, identical T and K (and identical ADG statistics).
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


@pytest.fixture(autouse=True)
def multi_kernel_path():
    """These tests cover the multi-kernel path (adg.cu + jp.cu) on every graph
    size: the one-kernel small-graph path (small.cu), which the default
    heuristic picks for small low-degree graphs, has its own file
    (test_gpu_small.py)."""
    pgc = pytest.importorskip("paper_2008_11321_b200")
    pgc.set_tuning("small_max_arcs", 0)
    yield
    pgc.set_tuning("small_max_arcs", 1 << 24)


def dev(g):
    pgc = pytest.importorskip("paper_2008_11321_b200")
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda() if g.nnz else torch.empty(0, dtype=torch.int32, device="cuda")
    return pgc, off, col


def run_gpu(g, num, den, seed):
    pgc, off, col = dev(g)
    rnd, color, T, K = pgc.color_jp_adg(off, col, num, den, seed)
    torch.cuda.synchronize()
    return rnd.cpu().numpy(), color.cpu().numpy(), T, K, pgc.last_stats()


def assert_parity(g, num, den, seed, stats=True):
    r_gpu, c_gpu, T, K, st = run_gpu(g, num, den, seed)
    r_or, st_or = O.adg(g, num, den)
    c_or, K_or = O.jp(g, r_or, seed)
    assert T == st_or["T"]
    bad = np.nonzero(r_gpu != r_or)[0]
    assert len(bad) == 0, f"round mismatch at {bad[:10]} gpu={r_gpu[bad[:10]]} cpu={r_or[bad[:10]]}"
    bad = np.nonzero(c_gpu != c_or)[0]
    assert len(bad) == 0, f"color mismatch at {bad[:10]} gpu={c_gpu[bad[:10]]} cpu={c_or[bad[:10]]}"
    assert K == K_or
    if stats:
        assert st["rounds"] == T and st["num_colors"] == K
        assert st["sum_active"] == st_or["sum_active"]
        assert st["cross_edges"] == st_or["cross_edges"]
        assert st["pred_arcs"] == g.m
    return T, K


def test_appendix_b_cases():
    cases = json.load(open(os.path.join(GOLDEN, "appendix_b.json")))["cases"]
    for c in cases:
        g = gg.from_edges(c["n"], c["edges"])
        for seed in (1, 2, 0xDEADBEEFCAFEF00D):
            T, K = assert_parity(g, c["eps"][0], c["eps"][1], seed)
            assert T == c["T"]


def test_zoo_all_graphs_up_to_5():
    # disjoint union of every labelled graph on <= 5 vertices
    edges, n = [], 0
    for k in range(1, 6):
        for es in all_graphs(k):
            edges += [(a + n, b + n) for a, b in es]
            n += k
    g = gg.from_edges(n, edges)
    for num, den in [(1, 100), (1, 10), (1, 2), (1, 1), (4294967295, 1)]:
        assert_parity(g, num, den, 7)


@pytest.mark.parametrize("seed", range(1, 9))
def test_random_er_rmat(seed):
    for g in (gg.er(3000, 15000 + 1000 * seed, seed), gg.rmat(8 + seed % 7, 8, seed=seed)):
        for num, den in [(1, 100), (1, 10), (1, 2)]:
            assert_parity(g, num, den, seed * 31 + 1)


def test_heavy_paths_cliques_and_hubs():
    # K_n: every vertex has up to n-1 preds -> heavy JP path; n > 2049 -> several color windows
    for n in (70, 300, 2100):
        g = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
        T, K = assert_parity(g, 1, 10, 3)
        assert T == 1 and K == n
    # star with a 5000-leaf hub -> heavy ADG UPDATE chunks
    g = gg.from_edges(5001, [(0, i) for i in range(1, 5001)])
    assert_parity(g, 1, 10, 3)
    # hub joined to a clique
    n = 400
    edges = [(i, j) for i in range(1, n) for j in range(i + 1, n)] + [(0, i) for i in range(1, 20000)]
    g = gg.from_edges(20000, edges)
    assert_parity(g, 1, 100, 5)


def test_edge_cases():
    pgc, off, col = dev(gg.from_edges(0, []))
    r, c, T, K = pgc.color_jp_adg(off, col, 1, 10, 1)
    assert T == 0 and K == 0 and r.numel() == 0
    for n in (1, 2, 33, 1000):
        assert_parity(gg.from_edges(n, []), 1, 10, 1)   # edgeless: one round, all color 1


@pytest.mark.parametrize("name", ["er", "rmat20", "grid"])
def test_config_parity(name):
    g = gg.config_graph(name)
    for num, den in gg.CONFIGS[name][1]:
        assert_parity(g, num, den, 1)


@pytest.mark.parametrize("name", ["rmat24", "cl"])
def test_config_parity_large(name):
    g = gg.config_graph(name)
    for num, den in gg.CONFIGS[name][1]:
        assert_parity(g, num, den, 1)


@pytest.fixture
def tuning():
    pgc = pytest.importorskip("paper_2008_11321_b200")
    touched = {}

    def set_(k, v):
        touched[k] = True
        pgc.set_tuning(k, v)
    yield set_
    defaults = {"core_max": 65535, "core_min_avg": 32, "core_min_n": 256, "core_ctas": 0,
                "core_arc_cap": 1 << 30, "core_arcs_per_cta": 2 << 20, "jp_heavy_warps": 4,
                "jp_heavy_sleep_max": 256, "jp_light_sleep_max": 8192,
                "heavy_degree": 128, "rounds_per_sync": 8, "jp_split_overlap": 1, "update_atom": 1, "fuse_init": 1, "top_list": 1,
                "core_tier2": 0, "jp_mega_pred": 2048, "jp_mega_chunk": 512,
                "itr_members_per_warp": 1, "jp_heavy_stripes": 1,
                "filter_ratio": 4, "chunk_arcs": 1024, "core_div": 32, "core_dmul": 20}
    for k in touched:
        pgc.set_tuning(k, defaults[k])


@pytest.mark.parametrize("ctas", [1, 2, 4, 8, 16])
def test_core_engine_cluster_sizes(ctas, tuning):
    """The cluster core engine (DSMEM color replicas) at every cluster size,
    forced onto graphs with a deep dense prefix, against the oracle."""
    tuning("core_ctas", ctas)
    tuning("core_min_n", 1)
    for g, (num, den) in ((gg.rmat(14, 16, seed=5), (1, 10)), (gg.rmat(13, 32, seed=8), (1, 100))):
        assert_parity(g, num, den, 11)
        st = pgc_stats()
        assert st["core_vertices"] > 0 and st["core_ctas"] >= 1


def test_core_engine_whole_graph_and_windows(tuning):
    """Every vertex in the core (min_avg 0) incl. K_n with > 2048 colors (several
    bitmap windows), and a core/bulk split right inside a round."""
    tuning("core_min_avg", 0)
    tuning("core_min_n", 1)
    n = 2100
    g = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    T, K = assert_parity(g, 1, 10, 3)
    assert K == n and pgc_stats()["core_vertices"] == n
    for cap in (1, 37, 1000):
        tuning("core_max", cap)
        assert_parity(gg.rmat(12, 16, seed=2), 1, 10, 4)
        assert pgc_stats()["core_vertices"] == cap


@pytest.mark.parametrize("mega", [(1024, 256), (1024, 1024), (4096, 2048), (0, 1024)])
def test_bulk_mega_vertices(mega, tuning):
    """Bulk vertices with more than jp_mega_pred preds are colored by one warp
    per pred chunk (the chunks OR their colors into one used-color set, the
    last one takes GetColor): no core (core_max 0), so K_2100's vertices of
    rank > 1024 are mega vertices and those of rank > 2048 find colors
    1..2048 all taken (the whole-list fallback from the second window); hubs
    and R-MAT under JP-ADG and JP-R; (0, .) = off."""
    pred, chunk = mega
    tuning("core_max", 0)
    tuning("jp_mega_pred", pred)
    tuning("jp_mega_chunk", chunk)
    n = 2100
    g = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    T, K = assert_parity(g, 1, 10, 3)
    assert K == n
    edges = [(i, j) for i in range(1, 400) for j in range(i + 1, 400)] + [(0, i) for i in range(1, 20000)]
    for g in (gg.from_edges(20000, edges), gg.rmat(15, 16, seed=2)):
        assert_parity(g, 1, 100, 5)
        pgc, off, col = dev(g)
        color, K = pgc.jp_baseline(off, col, "jp-r", 7)
        torch.cuda.synchronize()
        c_or, K_or = O.jp(g, np.zeros(g.n, dtype=np.int32), 7)
        assert np.array_equal(color.cpu().numpy(), c_or) and K == K_or


@pytest.mark.parametrize("stripes", [3, 8])
def test_bulk_heavy_ticket_stripes(stripes, tuning):
    """The heavy list dealt round-robin to several ticket counters (each
    stripe handed out in priority order): JP-ADG with and without the core,
    JP-R with mega vertices."""
    tuning("jp_heavy_stripes", stripes)
    g = gg.rmat(15, 16, seed=2)
    assert_parity(g, 1, 10, 5)
    tuning("core_max", 0)
    assert_parity(g, 1, 100, 6)
    n = 2100
    gk = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    for h in (g, gk):
        pgc, off, col = dev(h)
        color, K = pgc.jp_baseline(off, col, "jp-r", 7)
        torch.cuda.synchronize()
        c_or, K_or = O.jp(h, np.zeros(h.n, dtype=np.int32), 7)
        assert np.array_equal(color.cpu().numpy(), c_or) and K == K_or


def test_core_engine_tier2(tuning):
    """The second cluster pass (tier 2: int32 codes, tier-1 pred colors read
    from color[]) after a capped tier 1, forked and serial, with J."""
    for split in (1, 0):
        tuning("jp_split_overlap", split)
        for cap, t2 in ((1000, 2000), (300, 65535), (4096, 1)):
            tuning("core_max", cap)
            tuning("core_tier2", t2)
            tuning("core_min_n", 1)
            tuning("core_min_avg", 0)
            for g in (gg.rmat(14, 16, seed=5), gg.rmat(13, 32, seed=8)):
                assert_parity(g, 1, 10, 11)
                st = pgc_stats()
                assert st["core_vertices"] == min(cap + t2, g.n - int((g.degrees() == 0).sum()))
    pgc = pytest.importorskip("paper_2008_11321_b200")
    g = gg.rmat(14, 16, seed=5)
    _, off, col = dev(g)
    (rnd, color, T, K), J = _levels_gpu(pgc.color_jp_adg, off, col, 1, 10, 3)
    r_or, _ = O.adg(g, 1, 10)
    _, _, _, J_or = O.jp(g, r_or, 3, levels=True)
    assert J == J_or


def pgc_stats():
    import paper_2008_11321_b200 as pgc
    return pgc.last_stats()


def test_adg_order_only_and_jp_generic_keys():
    g = gg.rmat(13, 8, seed=4)
    pgc, off, col = dev(g)
    for num, den in [(1, 100), (1, 2)]:
        rnd, T = pgc.adg_order(off, col, num, den)
        r_or, st = O.adg(g, num, den)
        assert T == st["T"] and np.array_equal(rnd.cpu().numpy(), r_or)
        assert pgc.last_stats()["cross_edges"] == st["cross_edges"]
    seed = 11
    keys = {
        "adg": torch.from_numpy(O.adg(g, 1, 10)[0]).cuda(),
        "const(JP-R)": torch.full((g.n,), 5, dtype=torch.int32, device="cuda"),
        "degree(JP-LF)": torch.from_numpy(g.degrees().astype(np.int32)).cuda(),
        "negative": torch.from_numpy(-(np.arange(g.n) % 97).astype(np.int32)).cuda(),
    }
    for name, key in keys.items():
        color, K = pgc.jp_color(off, col, key, seed)
        c_or, K_or = O.jp(g, key.cpu().numpy(), seed)
        assert K == K_or and np.array_equal(color.cpu().numpy(), c_or), name
        assert pgc.last_stats()["pred_arcs"] == g.m


def test_jp_key_range_error():
    g = gg.er(100, 300, 1)
    pgc, off, col = dev(g)
    key = torch.zeros(g.n, dtype=torch.int32, device="cuda")
    key[0] = 2**31 - 1
    key[1] = -(2**31)
    with pytest.raises(pgc.PGCError) as e:
        pgc.jp_color(off, col, key, 1)
    assert e.value.code == pgc.PGC_EINVAL


def test_filtered_update_chunk_and_ratio_sweep(tuning):
    """The filtered late-round UPDATE (k_update_heavy_f; Alg. 1 UPDATE,
    PAPER.md:692-696, with the fused JP Part 1) against the oracle through
    JP-ADG, ADG only and JP-ADG-O: 256- and 300-arc chunks give ragged last
    steps and many chunk changes per warp, filter_ratio 1 / 2 start the filter
    in an earlier round (many hits per step)."""
    for hd, chunk, ratio in ((128, 1024, 4), (128, 256, 1), (160, 300, 2)):
        tuning("heavy_degree", hd)
        tuning("chunk_arcs", chunk)
        tuning("filter_ratio", ratio)
        for g, (num, den) in ((gg.rmat(15, 16, seed=4), (1, 10)), (gg.rmat(13, 32, seed=6), (1, 100)),
                              (gg.chung_lu(1 << 14, 32.0, 2.1, 1000.0, seed=3), (1, 2))):
            assert_parity(g, num, den, 5)
            pgc, off, col = dev(g)
            rnd, T = pgc.adg_order(off, col, num, den)
            r_or, st_or = O.adg(g, num, den)
            assert T == st_or["T"] and np.array_equal(rnd.cpu().numpy(), r_or)
            assert_parity_o(g, num, den)


def test_hub_chunk_descriptors(tuning):
    """Vertices with more than 8 edge chunks get one descriptor in the selection
    and their chunk records from k_round_aux (a warp per hub): hubs of degree
    2 100 .. 60 000 on a sparse background, removed in late rounds (UPDATE,
    PAPER.md:692-696), through JP-ADG, ADG push / pull and JP-ADG-M, with 256-
    and 1024-arc chunks (9 chunks = the first descriptor, a ragged last chunk)."""
    rng = np.random.default_rng(7)
    n = 70000
    edges = set()
    for hub, deg in ((0, 60000), (1, 2305), (2, 2100), (3, 9217), (4, 30001)):
        for u in rng.choice(np.arange(5, n), size=deg, replace=False):
            edges.add((hub, int(u)))
    for a, b in rng.integers(5, n, size=(150000, 2)):
        if a != b:
            edges.add((int(min(a, b)), int(max(a, b))))
    edges.update({(0, 1), (0, 2), (1, 3), (2, 4), (3, 4)})
    g = gg.from_edges(n, sorted(edges))
    for chunk in (256, 1024):
        tuning("chunk_arcs", chunk)
        for num, den in ((1, 10), (1, 2)):
            assert_parity(g, num, den, 3)
            assert_parity_pull(g, num, den)
        assert_parity_m(g, 3)


def test_determinism_across_tuning(tuning):
    g = gg.rmat(14, 16, seed=2)
    pgc, off, col = dev(g)
    ref = None
    for hd, rps, core, hw, sleep, ovl, atom in ((128, 1, 0, 1, 0, 1, 1), (200, 3, 65535, 2, 64, 0, 0),
                                                (1024, 8, 500, 4, 8192, 1, 0),
                                                (1 << 20, 8, 65535, 4, 2048, 1, 1),
                                                (128, 2, 0, 3, 100000, 0, 1)):
        tuning("jp_split_overlap", ovl)
        tuning("update_atom", atom)
        tuning("fuse_init", atom ^ ovl ^ 1)
        tuning("top_list", hw & 1)
        tuning("heavy_degree", hd)
        tuning("rounds_per_sync", rps)
        tuning("core_max", core)
        tuning("jp_heavy_warps", hw)
        tuning("jp_heavy_sleep_max", sleep)
        tuning("jp_light_sleep_max", sleep)
        for _ in range(2):
            r, c, T, K = pgc.color_jp_adg(off, col, 1, 10, 9)
            out = (r.cpu().numpy(), c.cpu().numpy(), T, K)
            if ref is None:
                ref = out
            assert np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1])
            assert out[2:] == ref[2:]
    r_or, _ = O.adg(g, 1, 10)
    c_or, _ = O.jp(g, r_or, 9)
    assert np.array_equal(ref[0], r_or) and np.array_equal(ref[1], c_or)


def test_host_api_matches_device_api():
    g = gg.rmat(12, 16, seed=6)
    pgc, off, col = dev(g)
    r_d, c_d, T_d, K_d = pgc.color_jp_adg(off, col, 1, 10, 3)
    h_off = torch.from_numpy(g.off).pin_memory()
    h_col = torch.from_numpy(g.col).pin_memory()
    h_r = torch.empty(g.n, dtype=torch.int32).pin_memory()
    h_c = torch.empty(g.n, dtype=torch.int32).pin_memory()
    T, K = pgc.color_jp_adg_host(h_off, h_col, 1, 10, 3, h_r, h_c)
    assert (T, K) == (T_d, K_d)
    assert torch.equal(h_r, r_d.cpu()) and torch.equal(h_c, c_d.cpu())


def test_check_graph():
    g = gg.rmat(10, 8, seed=1)
    pgc, off, col = dev(g)
    pgc.check_graph(off, col)
    bad = col.clone()
    # break symmetry: redirect one arc of the first nonempty row
    v = int(np.nonzero(g.degrees())[0][0])
    e = int(g.off[v])
    bad[e] = (bad[e] + 1) % g.n if int(bad[e] + 1) % g.n != v else (bad[e] + 2) % g.n
    with pytest.raises(pgc.PGCError) as ei:
        pgc.check_graph(off, bad)
    assert ei.value.code == pgc.PGC_EINVAL


def test_timing_stats():
    g = gg.rmat(12, 16, seed=6)
    pgc, off, col = dev(g)
    pgc.set_tuning("timing", 1)
    try:
        pgc.color_jp_adg(off, col, 1, 10, 3)
        st = pgc.last_stats()
        for k in ("t_select_ms", "t_update_ms", "t_order_ms", "t_jp_ms", "t_total_ms"):
            assert st[k] > 0, k
        parts = (st["t_select_ms"] + st["t_update_ms"] + st["t_adg_other_ms"] + st["t_order_ms"]
                 + st["t_core_ms"] + st["t_jp_ms"])
        assert parts <= st["t_total_ms"] * 1.01
        assert st["kernel_launches"] > 10 and st["host_syncs"] >= 2
    finally:
        pgc.set_tuning("timing", 0)


# ------------------------------------------------------------ ADG-M (NEXT-3) --
def assert_parity_m(g, seed):
    """JP-ADG-M through the C ABI against the ADG-M oracle + the JP oracle."""
    pgc, off, col = dev(g)
    rnd, color, T, K = pgc.color_jp_adg_m(off, col, seed)
    torch.cuda.synchronize()
    st = pgc.last_stats()
    r_gpu, c_gpu = rnd.cpu().numpy(), color.cpu().numpy()
    r_or, st_or = O.adg_m(g)
    c_or, K_or = O.jp(g, r_or, seed)
    assert T == st_or["T"] == (g.n.bit_length() if g.n else 0)
    bad = np.nonzero(r_gpu != r_or)[0]
    assert len(bad) == 0, f"ADG-M round mismatch at {bad[:10]} gpu={r_gpu[bad[:10]]} cpu={r_or[bad[:10]]}"
    bad = np.nonzero(c_gpu != c_or)[0]
    assert len(bad) == 0, f"color mismatch at {bad[:10]} gpu={c_gpu[bad[:10]]} cpu={c_or[bad[:10]]}"
    assert K == K_or
    assert st["sum_active"] == st_or["sum_active"] and st["cross_edges"] == st_or["cross_edges"]
    # ADG-M alone gives the same rounds
    r2, T2 = pgc.adg_m_order(off, col)
    torch.cuda.synchronize()
    assert T2 == T and np.array_equal(r2.cpu().numpy(), r_or)
    return T, K


def test_adg_m_hand_examples_and_small_graphs():
    for c in json.load(open(os.path.join(GOLDEN, "adg_m_examples.json")))["cases"]:
        g = gg.from_edges(c["n"], c["edges"])
        T, K = assert_parity_m(g, 1)
        assert T == c["T"]
    for n in range(0, 6):
        edges_all = list(all_graphs(n))
        # disjoint union of every graph on n vertices (one GPU call)
        es, base = [], 0
        for edges in edges_all:
            es += [(a + base, b + base) for a, b in edges]
            base += n
        assert_parity_m(gg.from_edges(base, es), 3)


@pytest.mark.parametrize("name", ["er", "rmat", "grid", "clique", "edgeless"])
def test_adg_m_random(name):
    g = {"er": lambda: gg.er(20000, 160000, 5), "rmat": lambda: gg.rmat(15, 16, seed=2),
         "grid": lambda: gg.grid(256, seed=4),
         "clique": lambda: gg.from_edges(300, [(i, j) for i in range(300) for j in range(i + 1, 300)]),
         "edgeless": lambda: gg.from_edges(1000, [])}[name]()
    for seed in (1, 9):
        assert_parity_m(g, seed)


@pytest.mark.parametrize("cfg", ["rmat20", "rmat24"])
def test_adg_m_full_size(cfg):
    g = gg.config_graph(cfg)
    assert_parity_m(g, 1)


# ------------------------------------------------------------ ADG-O (NEXT-1) --
def assert_parity_o(g, num, den):
    """JP-ADG-O through the C ABI against the ADG-O oracle + JP for rho."""
    pgc, off, col = dev(g)
    rnd, color, T, K = pgc.color_jp_adg_o(off, col, num, den)
    torch.cuda.synchronize()
    st = pgc.last_stats()
    r_gpu, c_gpu = rnd.cpu().numpy(), color.cpu().numpy()
    r_or, rho, rank, drem, T_or = O.adg_o(g, num, den)
    c_or, K_or = O.jp_rho(g, rho)
    assert T == T_or
    bad = np.nonzero(r_gpu != r_or)[0]
    assert len(bad) == 0, f"round mismatch at {bad[:10]}"
    bad = np.nonzero(c_gpu != c_or)[0]
    assert len(bad) == 0, f"ADG-O color mismatch at {bad[:10]} gpu={c_gpu[bad[:10]]} cpu={c_or[bad[:10]]}"
    assert K == K_or
    assert st["pred_arcs"] == g.m   # every edge gives exactly one pred (a total order)
    return T, K


def test_adg_o_hand_examples_and_small_graphs():
    for c in json.load(open(os.path.join(GOLDEN, "adg_o_examples.json")))["cases"]:
        g = gg.from_edges(c["n"], c["edges"])
        T, K = assert_parity_o(g, *c["eps"])
        assert K == c["K"]
    for n in range(0, 6):
        es, base = [], 0
        for edges in all_graphs(n):
            es += [(a + base, b + base) for a, b in edges]
            base += n
        for num, den in [(1, 10), (1, 2)]:
            assert_parity_o(gg.from_edges(base, es), num, den)


@pytest.mark.parametrize("name", ["er", "rmat", "grid", "clique", "edgeless"])
def test_adg_o_random(name):
    g = {"er": lambda: gg.er(20000, 160000, 5), "rmat": lambda: gg.rmat(15, 16, seed=2),
         "grid": lambda: gg.grid(256, seed=4),
         "clique": lambda: gg.from_edges(300, [(i, j) for i in range(300) for j in range(i + 1, 300)]),
         "edgeless": lambda: gg.from_edges(1000, [])}[name]()
    for num, den in [(1, 100), (1, 10), (1, 2)]:
        assert_parity_o(g, num, den)


@pytest.mark.parametrize("cfg", ["rmat20", "rmat24"])
def test_adg_o_full_size(cfg):
    g = gg.config_graph(cfg)
    assert_parity_o(g, *gg.CONFIGS[cfg][1][0])


# ------------------------------------------------ JP baselines (NEXT-4) -------
@pytest.mark.parametrize("kind", ["jp-r", "jp-ff", "jp-lf", "jp-llf"])
def test_jp_baselines(kind):
    import math
    for g, seed in [(gg.from_edges(5, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)]), 1),
                    (gg.er(20000, 160000, 5), 2), (gg.rmat(15, 16, seed=2), 3), (gg.grid(256, seed=4), 4),
                    (gg.config_graph("rmat20"), 1)]:
        pgc, off, col = dev(g)
        color, K = pgc.jp_baseline(off, col, kind, seed)
        torch.cuda.synchronize()
        deg = g.degrees()
        key = {"jp-r": np.zeros(g.n), "jp-ff": -np.arange(g.n), "jp-lf": deg,
               "jp-llf": np.array([math.ceil(math.log2(d)) if d > 1 else 0 for d in deg])}[kind]
        c_or, K_or = O.jp(g, key.astype(np.int32), seed)
        bad = np.nonzero(color.cpu().numpy() != c_or)[0]
        assert len(bad) == 0, f"{kind}: color mismatch at {bad[:10]}"
        assert K == K_or


# ------------------------------------------------ DEC-ADG-ITR (NEXT-2) --------
def assert_parity_dec(g, num, den, seed):
    pgc, off, col = dev(g)
    rnd, color, T, K = pgc.color_dec_adg_itr(off, col, num, den, seed)
    torch.cuda.synchronize()
    st = pgc.last_stats()
    r_or, st_or = O.adg(g, num, den)
    c_or, K_or, passes = O.dec_adg_itr(g, r_or, seed)
    assert T == st_or["T"] and np.array_equal(rnd.cpu().numpy(), r_or)
    bad = np.nonzero(color.cpu().numpy() != c_or)[0]
    assert len(bad) == 0, f"DEC-ADG-ITR color mismatch at {bad[:10]} gpu={color.cpu().numpy()[bad[:10]]} cpu={c_or[bad[:10]]}"
    assert K == K_or
    return T, K


def test_dec_adg_itr_small_graphs():
    for n in range(0, 6):
        es, base = [], 0
        for edges in all_graphs(n):
            es += [(a + base, b + base) for a, b in edges]
            base += n
        for num, den in [(1, 10), (1, 2)]:
            for seed in (1, 2):
                assert_parity_dec(gg.from_edges(base, es), num, den, seed)
    n = 40
    assert_parity_dec(gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)]), 1, 10, 3)


@pytest.mark.parametrize("name", ["er", "rmat", "grid", "edgeless"])
def test_dec_adg_itr_random(name):
    g = {"er": lambda: gg.er(20000, 160000, 5), "rmat": lambda: gg.rmat(15, 16, seed=2),
         "grid": lambda: gg.grid(256, seed=4), "edgeless": lambda: gg.from_edges(1000, [])}[name]()
    for num, den in [(1, 100), (1, 10), (1, 2)]:
        assert_parity_dec(g, num, den, 7)


@pytest.mark.parametrize("mpw", [4, 64])
def test_dec_adg_itr_pass_grid_sizes(mpw, tuning):
    """The SIM-COL pass grid sized at 4 and 64 partition members per warp (one
    block for most partitions: the grid barrier among one block), on a clique
    (one vertex fixed per pass) and R-MAT."""
    tuning("itr_members_per_warp", mpw)
    n = 300
    g = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    T, K = assert_parity_dec(g, 1, 10, 3)
    assert K == n
    assert_parity_dec(gg.rmat(15, 16, seed=2), 1, 10, 7)


def test_dec_adg_itr_rmat20():
    assert_parity_dec(gg.config_graph("rmat20"), 1, 10, 1)


def test_dec_adg_itr_and_baselines_rmat24():
    """The headline graph (R-MAT 24, 520 M arcs) on DEC-ADG-ITR and on the JP
    baselines without a dense priority prefix (JP-R, JP-FF: no core, long
    chains in the bulk) and with one (JP-LLF)."""
    import math
    g = gg.config_graph("rmat24")
    assert_parity_dec(g, 1, 10, 1)
    pgc, off, col = dev(g)
    deg = g.degrees()
    for kind in ("jp-r", "jp-ff", "jp-llf"):
        color, K = pgc.jp_baseline(off, col, kind, 1)
        torch.cuda.synchronize()
        key = {"jp-r": np.zeros(g.n), "jp-ff": -np.arange(g.n),
               "jp-llf": np.ceil(np.log2(np.maximum(deg, 1)))}[kind]
        c_or, K_or = O.jp(g, key.astype(np.int32), 1)
        bad = np.nonzero(color.cpu().numpy() != c_or)[0]
        assert len(bad) == 0, f"{kind}: color mismatch at {bad[:10]}"
        assert K == K_or


# ------------------------------------- next rows on the other full-size configs --
@pytest.mark.parametrize("cfg", ["cl", "grid"])
def test_next_rows_full_size(cfg):
    """ADG-O, ADG-M and DEC-ADG-ITR at full size on the heavy-hub Chung-Lu graph
    and the low-degree grid (many ADG rounds)."""
    g = gg.config_graph(cfg)
    eps = gg.CONFIGS[cfg][1]
    assert_parity_o(g, *eps[0])
    assert_parity_m(g, 5)
    assert_parity_dec(g, *eps[-1], 3)


# ------------------------------------------------ repeat / stress -------------
def test_repeat_runs_are_identical_and_never_stall():
    """The dataflow kernels are schedule-dependent inside; the results must not
    be.  Repeats of every entry point on one graph, with a short watchdog (a
    stall would surface as PGC_EINTERNAL, not a hang)."""
    pgc = pytest.importorskip("paper_2008_11321_b200")
    g = gg.rmat(17, 16, seed=9)
    _, off, col = dev(g)
    pgc.set_tuning("jp_watchdog_ms", 5000)
    try:
        ref = None
        for rep in range(12):
            out = []
            r, c, T, K = pgc.color_jp_adg(off, col, 1, 10, 4)
            out += [r.cpu().numpy(), c.cpu().numpy()]
            r, c, T, K = pgc.color_jp_adg_o(off, col, 1, 10)
            out += [c.cpu().numpy()]
            for kind in ("jp-r", "jp-lf"):
                c, K = pgc.jp_baseline(off, col, kind, 4)
                out += [c.cpu().numpy()]
            r, c, T, K = pgc.color_dec_adg_itr(off, col, 1, 10, 4)
            out += [c.cpu().numpy()]
            if ref is None:
                ref = out
            else:
                assert all(np.array_equal(x, y) for x, y in zip(out, ref)), f"repeat {rep} differs"
    finally:
        pgc.set_tuning("jp_watchdog_ms", 20000)


# ------------------------------------------ pull (CREW) UPDATE (NEXT-4) -------
def assert_parity_pull(g, num, den):
    """pgc_adg_order_mode with PGC_UPDATE_PULL (and PUSH) against the ADG oracle:
    identical rounds and identical round statistics (the decrements are the
    same integers)."""
    pgc, off, col = dev(g)
    r_or, st_or = O.adg(g, num, den)
    for upd in ("pull", "push"):
        rnd, T = pgc.adg_order(off, col, num, den, update=upd)
        torch.cuda.synchronize()
        st = pgc.last_stats()
        assert T == st_or["T"], upd
        bad = np.nonzero(rnd.cpu().numpy() != r_or)[0]
        assert len(bad) == 0, f"{upd} round mismatch at {bad[:10]}"
        assert st["sum_active"] == st_or["sum_active"], upd
        assert st["cross_edges"] == st_or["cross_edges"], upd
    return st_or["T"]


def test_adg_pull_small_graphs():
    for c in json.load(open(os.path.join(GOLDEN, "appendix_b.json")))["cases"]:
        assert assert_parity_pull(gg.from_edges(c["n"], c["edges"]), *c["eps"]) == c["T"]
    edges, n = [], 0
    for k in range(1, 6):
        for es in all_graphs(k):
            edges += [(a + n, b + n) for a, b in es]
            n += k
    g = gg.from_edges(n, edges)
    for num, den in [(1, 100), (1, 10), (1, 2), (4294967295, 1)]:
        assert_parity_pull(g, num, den)
    pgc, off, col = dev(gg.from_edges(0, []))
    assert pgc.adg_order(off, col, 1, 10, update="pull")[1] == 0


def test_adg_pull_hubs_and_random():
    # surviving hubs: a 5000-leaf star (the hub survives round 1 and is a
    # chunked record of the pull UPDATE) and a hub joined to a clique
    assert_parity_pull(gg.from_edges(5001, [(0, i) for i in range(1, 5001)]), 1, 10)
    n = 400
    edges = [(i, j) for i in range(1, n) for j in range(i + 1, n)] + [(0, i) for i in range(1, 20000)]
    assert_parity_pull(gg.from_edges(20000, edges), 1, 100)
    for seed in range(1, 5):
        for g in (gg.er(3000, 15000 + 1000 * seed, seed), gg.rmat(10 + seed, 16, seed=seed)):
            for num, den in [(1, 100), (1, 10), (1, 2)]:
                assert_parity_pull(g, num, den)


@pytest.mark.parametrize("cfg", ["rmat20", "grid", "rmat24"])
def test_adg_pull_full_size(cfg):
    g = gg.config_graph(cfg)
    for num, den in gg.CONFIGS[cfg][1][-1:]:
        assert_parity_pull(g, num, den)


def test_more_than_255_rounds_every_entry_point():
    """Paths with eps < 1/(n-1) peel two ends per round (closed form pinned in
    test_oracle_pins): 500 / 501 rounds, past the one-byte round state's
    255, so the late rounds classify arcs from round[] (Arc::raw)."""
    for n in (1000, 1001):
        # P_n plus P_601, randomly relabelled (mean degree stays below 2)
        edges = [(i, i + 1) for i in range(n - 1)] + [(n + i, n + i + 1) for i in range(600)]
        perm = np.random.default_rng(n).permutation(n + 601)
        g = gg.from_edges(n + 601, [(int(perm[a]), int(perm[b])) for a, b in edges])
        den = 100 * n
        T = assert_parity_pull(g, 1, den)
        assert T > 255
        assert_parity(g, 1, den, 3)
        assert_parity_o(g, 1, den)
        assert_parity_dec(g, 1, den, 3)


def test_serialised_kernels_do_not_deadlock():
    """With every launch serialised (CUDA_LAUNCH_BLOCKING=1, as under a
    profiler) the core kernel cannot wait for the list rewrite running beside
    it: it must claim and rewrite the lists itself (claim protocol in jp.cu).
    A fresh process also exercises the first-call path (kernels loaded before
    the fork)."""
    import subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, 'tests')\n"
        "import numpy as np, torch\n"
        "import graphgen as gg, oracle as O, paper_2008_11321_b200 as pgc\n"
        "pgc.set_tuning('jp_watchdog_ms', 5000); pgc.set_tuning('small_max_arcs', 0)\n"
        "g = gg.rmat(15, 16, seed=6)\n"
        "off = torch.from_numpy(g.off).cuda(); col = torch.from_numpy(g.col).cuda()\n"
        "r, c, T, K = pgc.color_jp_adg(off, col, 1, 10, 5)\n"
        "assert pgc.last_stats()['core_vertices'] > 0\n"
        "r_or, _ = O.adg(g, 1, 10); c_or, K_or = O.jp(g, r_or, 5)\n"
        "assert np.array_equal(r.cpu().numpy(), r_or) and np.array_equal(c.cpu().numpy(), c_or)\n"
        "print('ok')\n")
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


# ---- J (JP levels, pgc_stats.jp_levels) against the oracle's level[] -------
def _levels_gpu(fn, *args):
    pgc = pytest.importorskip("paper_2008_11321_b200")
    pgc.set_tuning("levels", 1)
    try:
        out = fn(*args)
        torch.cuda.synchronize()
        return out, pgc.last_stats()["jp_levels"]
    finally:
        pgc.set_tuning("levels", 0)


@pytest.mark.parametrize("name", ["er", "rmat20", "grid"])
def test_jp_levels_match_oracle(name):
    # J = 1 + the longest chain of higher-priority neighbours:
    # on rmat20 the core engine colors the top of the order (u16 lists), the bulk the rest
    g = gg.config_graph(name)
    pgc, off, col = dev(g)
    num, den = gg.CONFIGS[name][1][0]
    (rnd, color, T, K), J = _levels_gpu(pgc.color_jp_adg, off, col, num, den, 1)
    r_or, _ = O.adg(g, num, den)
    c_or, K_or, lvl, J_or = O.jp(g, r_or, 1, levels=True)
    assert np.array_equal(color.cpu().numpy(), c_or)
    assert J == J_or, (J, J_or)
    # the levels pass changes no result and is off by default
    pgc.color_jp_adg(off, col, num, den, 1)
    assert pgc.last_stats()["jp_levels"] == 0


def test_jp_levels_small_cases():
    pgc = pytest.importorskip("paper_2008_11321_b200")
    # clique K_n: J = n; star: 2; edgeless: 1; path at eps 1/2
    for g in (gg.from_edges(50, [(i, j) for i in range(50) for j in range(i + 1, 50)]),
              gg.from_edges(6, [(0, i) for i in range(1, 6)]),
              gg.from_edges(5, []),
              gg.from_edges(9, [(i, i + 1) for i in range(8)]),
              gg.rmat(12, 16, seed=5)):
        _, off, col = dev(g)
        for num, den in [(1, 10), (1, 2)]:
            (rnd, color, T, K), J = _levels_gpu(pgc.color_jp_adg, off, col, num, den, 3)
            r_or, _ = O.adg(g, num, den)
            _, _, _, J_or = O.jp(g, r_or, 3, levels=True)
            assert J == J_or


def test_jp_levels_generic_key():
    # pgc_jp_color with JP-R (constant key) and the baselines: same J as the oracle
    g = gg.rmat(13, 8, seed=9)
    pgc, off, col = dev(g)
    key = torch.zeros(g.n, dtype=torch.int32, device="cuda")
    (color, K), J = _levels_gpu(pgc.jp_color, off, col, key, 11)
    _, _, _, J_or = O.jp(g, np.zeros(g.n, dtype=np.int32), 11, levels=True)
    assert J == J_or


def test_second_device_if_present():
    # per-device attributes, occupancy and side streams: one process driving two GPUs
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU")
    g = gg.rmat(14, 16, seed=2)
    pgc = pytest.importorskip("paper_2008_11321_b200")
    r_or, _ = O.adg(g, 1, 10)
    c_or, _ = O.jp(g, r_or, 1)
    for d in (0, 1, 0):
        off = torch.from_numpy(g.off).to(f"cuda:{d}")
        col = torch.from_numpy(g.col).to(f"cuda:{d}")
        rnd, color, T, K = pgc.color_jp_adg(off, col, 1, 10, 1)
        assert np.array_equal(color.cpu().numpy(), c_or)
