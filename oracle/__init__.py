"""Sequential CPU oracle for JP-ADG -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2008_11321_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``oracle.c`` (plain single-threaded C, each
function citing PAPER.md); this file only marshals arguments via ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o", _SO, _SRC])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp, i64, u64, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32
        lib.orc_splitmix64.restype = u64
        lib.orc_splitmix64.argtypes = [u64]
        lib.orc_adg.restype = ctypes.c_int
        lib.orc_adg.argtypes = [i64, vp, vp, u32, u32, vp, vp, i64, vp, vp, vp]
        lib.orc_adg_o.restype = ctypes.c_int
        lib.orc_adg_o.argtypes = [i64, vp, vp, u32, u32, vp, vp, vp, vp]
        lib.orc_jp_rho.restype = ctypes.c_int
        lib.orc_jp_rho.argtypes = [i64, vp, vp, vp, vp]
        lib.orc_dec_adg_itr.restype = ctypes.c_int
        lib.orc_dec_adg_itr.argtypes = [i64, vp, vp, vp, ctypes.c_int32, u64, vp, vp]
        lib.orc_adg_m.restype = ctypes.c_int
        lib.orc_adg_m.argtypes = [i64, vp, vp, vp, vp]
        lib.orc_jp.restype = ctypes.c_int
        lib.orc_jp.argtypes = [i64, vp, vp, vp, u64, vp, vp, vp]
        lib.orc_degeneracy.restype = i64
        lib.orc_degeneracy.argtypes = [i64, vp, vp]
        lib.orc_brute_chi.restype = ctypes.c_int
        lib.orc_brute_chi.argtypes = [i64, vp, vp]
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data if a is not None and a.size > 0 else None


def _csr(g):
    off = np.ascontiguousarray(g.off, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int32)
    return off, col


def splitmix64(x: int) -> int:
    return int(_load().orc_splitmix64(x & 0xFFFFFFFFFFFFFFFF))


def adg(g, num: int, den: int, per_round: bool = False):
    """ADG rounds (Alg. 1).  Returns (round int32[n], stats dict)."""
    off, col = _csr(g)
    n = g.n
    rnd = np.zeros(n, dtype=np.int32)
    st = np.zeros(4, dtype=np.int64)
    cap = 1 << 16 if per_round else 0
    pn = np.zeros(cap, dtype=np.int64) if per_round else None
    ps = np.zeros(cap, dtype=np.int64) if per_round else None
    pr = np.zeros(cap, dtype=np.int64) if per_round else None
    T = _load().orc_adg(n, _p(off), _p(col), num, den, _p(rnd), _p(st), cap, _p(pn), _p(ps), _p(pr))
    if T == -1:
        raise ValueError("oracle adg: bad arguments")
    if T < 0:
        raise RuntimeError("oracle adg: a round selected no vertex")
    stats = {"T": int(st[0]), "sum_active": int(st[1]), "cross_edges": int(st[2]),
             "all_decrements": int(st[3])}
    if per_round:
        stats["nU"] = pn[:T].copy()
        stats["S"] = ps[:T].copy()
        stats["nR"] = pr[:T].copy()
    return rnd, stats


def adg_o(g, num: int, den: int):
    """ADG-O.  Returns (round int32, rho int64, rank int64, drem int64, T)."""
    off, col = _csr(g)
    n = g.n
    rnd = np.zeros(n, dtype=np.int32)
    rho = np.zeros(n, dtype=np.int64)
    rank = np.zeros(n, dtype=np.int64)
    drem = np.zeros(n, dtype=np.int64)
    T = _load().orc_adg_o(n, _p(off), _p(col), num, den, _p(rnd), _p(rho), _p(rank), _p(drem))
    if T < 0:
        raise ValueError("oracle adg_o: bad arguments")
    return rnd, rho, rank, drem, int(T)


def jp_rho(g, rho):
    """JP colors for a total-order priority rho (int64, larger first).  Returns (color, K)."""
    off, col = _csr(g)
    rho = np.ascontiguousarray(rho, dtype=np.int64)
    color = np.zeros(g.n, dtype=np.int32)
    K = _load().orc_jp_rho(g.n, _p(off), _p(col), _p(rho), _p(color))
    if K < 0:
        raise ValueError("oracle jp_rho: bad arguments")
    return color, int(K)


def dec_adg_itr(g, rnd, seed: int):
    """DEC-ADG-ITR colors for ADG rounds rnd.  Returns (color, K, passes)."""
    off, col = _csr(g)
    rnd = np.ascontiguousarray(rnd, dtype=np.int32)
    color = np.zeros(g.n, dtype=np.int32)
    passes = ctypes.c_int64(0)
    T = int(rnd.max()) if g.n else 0
    K = _load().orc_dec_adg_itr(g.n, _p(off), _p(col), _p(rnd), T, seed & 0xFFFFFFFFFFFFFFFF,
                                _p(color), ctypes.addressof(passes))
    if K < 0:
        raise ValueError("oracle dec_adg_itr: bad arguments")
    return color, int(K), int(passes.value)


def adg_m(g):
    """ADG-M rounds (median threshold).  Returns (round int32[n], stats)."""
    off, col = _csr(g)
    rnd = np.zeros(g.n, dtype=np.int32)
    st = np.zeros(3, dtype=np.int64)
    T = _load().orc_adg_m(g.n, _p(off), _p(col), _p(rnd), _p(st))
    if T < 0:
        raise ValueError("oracle adg_m: bad arguments")
    return rnd, {"T": int(st[0]), "sum_active": int(st[1]), "cross_edges": int(st[2])}


def jp(g, rnd, seed: int, levels: bool = False):
    """JP colors for priority <round, splitmix64(seed^v)>.  Returns (color, K[, level, J])."""
    off, col = _csr(g)
    rnd = np.ascontiguousarray(rnd, dtype=np.int32)
    color = np.zeros(g.n, dtype=np.int32)
    lvl = np.zeros(g.n, dtype=np.int32) if levels else None
    J = ctypes.c_int64(0)
    K = _load().orc_jp(g.n, _p(off), _p(col), _p(rnd), seed & 0xFFFFFFFFFFFFFFFF, _p(color),
                       _p(lvl), ctypes.addressof(J))
    if K < 0:
        raise ValueError("oracle jp: bad arguments")
    if levels:
        return color, int(K), lvl, int(J.value)
    return color, int(K)


def jp_adg(g, num: int, den: int, seed: int):
    """Whole method: (round, color, T, K, adg stats)."""
    rnd, st = adg(g, num, den)
    color, K = jp(g, rnd, seed)
    return rnd, color, st["T"], K, st


def degeneracy(g) -> int:
    off, col = _csr(g)
    return int(_load().orc_degeneracy(g.n, _p(off), _p(col)))


def brute_chi(g) -> int:
    off, col = _csr(g)
    r = _load().orc_brute_chi(g.n, _p(off), _p(col))
    if r < 0:
        raise ValueError("brute_chi: n > 16")
    return int(r)
