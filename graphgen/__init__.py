"""Seeded synthetic graph inputs shared by the oracle and the CUDA path.

Input harness only: this package holds no arithmetic of the method (no ADG,
no priority hash, no coloring).  The generators live in ``graphgen.c``
(C + OpenMP, counter-based RNG, thread-count independent) and are reached
through ctypes.  Recipes: BASELINE.json ``configs`` / SURVEY.md §8(d); the
exact recipe per config is restated in DESIGN.md ("Input recipe").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgraphgen.so")
_SRC = os.path.join(_HERE, "graphgen.c")


def build(force: bool = False) -> str:
    """Compile libgraphgen.so in-tree (gcc, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared",
                               "-std=c11", "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp = ctypes.c_void_p
        i64, u64, dbl, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int
        lib.gg_er.restype = vp
        lib.gg_er.argtypes = [i64, i64, u64]
        lib.gg_rmat.restype = vp
        lib.gg_rmat.argtypes = [i32, i64, dbl, dbl, dbl, u64]
        lib.gg_grid.restype = vp
        lib.gg_grid.argtypes = [i64, dbl, dbl, u64]
        lib.gg_chung_lu.restype = vp
        lib.gg_chung_lu.argtypes = [i64, dbl, dbl, dbl, u64]
        lib.gg_from_edges.restype = vp
        lib.gg_from_edges.argtypes = [i64, i64, vp, vp]
        lib.gg_n.restype = i64
        lib.gg_n.argtypes = [vp]
        lib.gg_nnz.restype = i64
        lib.gg_nnz.argtypes = [vp]
        lib.gg_take.restype = None
        lib.gg_take.argtypes = [vp, vp, vp]
        lib.gg_free.restype = None
        lib.gg_free.argtypes = [vp]
        _lib = lib
    return _lib


@dataclass
class Graph:
    """Undirected simple graph in CSR: int64 offsets[n+1], int32 cols[nnz]."""
    n: int
    off: np.ndarray
    col: np.ndarray
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.off[-1]) if self.n >= 0 else 0

    @property
    def m(self) -> int:
        return self.nnz // 2

    def degrees(self) -> np.ndarray:
        return np.diff(self.off)


def _take(h, name: str) -> Graph:
    lib = _load()
    n, nnz = lib.gg_n(h), lib.gg_nnz(h)
    off = np.empty(n + 1, dtype=np.int64)
    col = np.empty(max(nnz, 0), dtype=np.int32)
    lib.gg_take(h, off.ctypes.data, col.ctypes.data if nnz > 0 else None)
    lib.gg_free(h)
    return Graph(int(n), off, col, name)


def from_edges(n: int, edges, name: str = "") -> Graph:
    """CSR from an arbitrary undirected edge list (symmetrise, dedup, drop loops)."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    u = np.ascontiguousarray(e[:, 0].astype(np.int32))
    v = np.ascontiguousarray(e[:, 1].astype(np.int32))
    h = _load().gg_from_edges(n, len(u), u.ctypes.data if len(u) else None,
                              v.ctypes.data if len(v) else None)
    return _take(h, name)


def er(n: int, m: int, seed: int = 1) -> Graph:
    return _take(_load().gg_er(n, m, seed), f"er(n={n},m={m},seed={seed})")


def rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
         seed: int = 1) -> Graph:
    return _take(_load().gg_rmat(scale, edge_factor, a, b, c, seed),
                 f"rmat(scale={scale},ef={edge_factor},seed={seed})")


def grid(W: int = 2048, p_keep: float = 0.7, p_diag: float = 0.02, seed: int = 1) -> Graph:
    return _take(_load().gg_grid(W, p_keep, p_diag, seed), f"grid(W={W},seed={seed})")


def chung_lu(n: int = 1 << 23, mean_deg: float = 32.0, gamma: float = 2.1, wmax: float = 1e5,
             seed: int = 1) -> Graph:
    return _take(_load().gg_chung_lu(n, mean_deg, gamma, wmax, seed),
                 f"chung_lu(n={n},mean={mean_deg},gamma={gamma},seed={seed})")


# BASELINE.json configs: name -> (builder, [(eps_num, eps_den), ...])
CONFIGS = {
    "er":     (lambda: er(16384, 131072, 1), [(1, 10)]),
    "rmat20": (lambda: rmat(20, 16, seed=1), [(1, 100), (1, 10), (1, 2)]),
    "grid":   (lambda: grid(2048, 0.7, 0.02, seed=1), [(1, 10)]),
    "rmat24": (lambda: rmat(24, 16, seed=1), [(1, 10)]),
    "cl":     (lambda: chung_lu(1 << 23, 32.0, 2.1, 1e5, seed=1), [(1, 100), (1, 2)]),
}

_cache: dict = {}


def config_graph(name: str) -> Graph:
    if name not in _cache:
        g = CONFIGS[name][0]()
        g.name = name
        _cache[name] = g
    return _cache[name]
