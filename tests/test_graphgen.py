"""Input harness: CSR invariants and determinism of the seeded generators."""
import numpy as np
import pytest

import graphgen as gg


def csr_ok(g):
    off, col = g.off, g.col
    assert off[0] == 0 and (np.diff(off) >= 0).all() and off[-1] == len(col)
    if g.nnz == 0:
        return
    assert col.min() >= 0 and col.max() < g.n
    src = np.repeat(np.arange(g.n), np.diff(off))
    assert not (src == col).any(), "self-loop"
    # rows strictly ascending (sorted, no duplicates)
    same_row = src[1:] == src[:-1]
    assert (col[1:][same_row] > col[:-1][same_row]).all()
    # symmetric
    fwd = src.astype(np.int64) * g.n + col
    bwd = col.astype(np.int64) * g.n + src
    assert np.array_equal(np.sort(fwd), np.sort(bwd))


def test_from_edges_cleans():
    g = gg.from_edges(4, [(0, 1), (1, 0), (2, 2), (3, 1), (1, 3), (0, 1)])
    csr_ok(g)
    assert g.off.tolist() == [0, 1, 3, 3, 4] and g.col.tolist() == [1, 0, 3, 1]


def test_er_exact_m_and_deterministic():
    a = gg.er(16384, 131072, 1)
    b = gg.er(16384, 131072, 1)
    csr_ok(a)
    assert a.m == 131072 and a.n == 16384
    assert np.array_equal(a.col, b.col)
    c = gg.er(16384, 131072, 2)
    assert not np.array_equal(a.col, c.col)


def test_rmat_shape():
    g = gg.rmat(12, 8, seed=3)
    csr_ok(g)
    assert g.n == 4096
    d = g.degrees()
    assert d.max() > 20 * d.mean()           # skewed
    assert (d == 0).sum() > 0                 # isolated vertices are kept (Q12)
    assert np.array_equal(g.col, gg.rmat(12, 8, seed=3).col)


def test_grid_shape():
    g = gg.grid(128, seed=2)
    csr_ok(g)
    d = g.degrees()
    assert d.max() <= 8
    assert 2.4 < d.mean() < 3.3


def test_chung_lu_shape():
    g = gg.chung_lu(1 << 14, 32.0, 2.1, 1e3, seed=1)
    csr_ok(g)
    d = g.degrees()
    assert d.max() <= 2 * 1e3 + 50
    assert 20 < d.mean() < 33


def test_thread_count_independence():
    import subprocess, sys, os
    code = ("import graphgen as gg, hashlib; g = gg.rmat(12, 8, seed=9); "
            "print(hashlib.sha1(g.col.tobytes() + g.off.tobytes()).hexdigest())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = set()
    for t in ("1", "3"):
        env = dict(os.environ, OMP_NUM_THREADS=t, PYTHONPATH=root)
        outs.add(subprocess.check_output([sys.executable, "-c", code], env=env, cwd=root).strip())
    assert len(outs) == 1
