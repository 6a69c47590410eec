"""pgc -- B200-native JP-ADG graph coloring (arXiv 2008.11321), Python binding.

A thin ctypes layer over the C ABI in ``include/pgc.h`` (``libpgc.so``, built
in-tree from ``csrc/`` by ``_build.py``).  It only marshals arguments: every
step of ADG and JP runs in the library's CUDA kernels.  PyTorch supplies
device memory and the current stream.  There is no CPU fallback: importing
this package fails loudly when the extension is missing.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# PGC_LIB may point at another build of the same ABI (A/B experiments only)
SO_PATH = os.environ.get("PGC_LIB") or os.path.join(_HERE, "libpgc.so")

if not os.path.exists(SO_PATH):
    raise ImportError(f"libpgc.so not found at {SO_PATH}: build it with "
                      f"`python -m paper_2008_11321_b200._build` (nvcc, sm_100a). "
                      f"There is no CPU fallback.")

_lib = ctypes.CDLL(SO_PATH)

PGC_OK, PGC_EINVAL, PGC_EWORKSPACE, PGC_ECUDA, PGC_EINTERNAL = 0, 1, 2, 3, 4

EXPORTS = ["pgc_workspace_bytes", "pgc_adg_order", "pgc_adg_order_mode", "pgc_jp_color", "pgc_color_jp_adg",
           "pgc_adg_m_order", "pgc_color_jp_adg_m", "pgc_color_jp_adg_o", "pgc_jp_baseline",
           "pgc_color_dec_adg_itr",
           "pgc_host_workspace_bytes", "pgc_color_jp_adg_host", "pgc_check_graph",
           "pgc_last_stats", "pgc_last_error", "pgc_set_tuning", "pgc_version",
           "pgc_debug_set_trace"]


class Graph(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_offsets", ctypes.c_void_p), ("col_indices", ctypes.c_void_p)]


class Stats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int32), ("num_colors", ctypes.c_int32),
                ("sum_active", ctypes.c_int64), ("cross_edges", ctypes.c_int64),
                ("pred_arcs", ctypes.c_int64), ("core_vertices", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int32), ("host_syncs", ctypes.c_int32),
                ("core_ctas", ctypes.c_int32), ("sim_col_passes", ctypes.c_int32),
                ("jp_levels", ctypes.c_int32),
                ("t_select_ms", ctypes.c_float), ("t_update_ms", ctypes.c_float),
                ("t_adg_other_ms", ctypes.c_float), ("t_order_ms", ctypes.c_float),
                ("t_core_ms", ctypes.c_float), ("t_jp_ms", ctypes.c_float),
                ("t_total_ms", ctypes.c_float), ("small_path", ctypes.c_int32)]


_vp, _i64, _u32, _u64, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t
_i32p = ctypes.POINTER(ctypes.c_int32)
_GP = ctypes.POINTER(Graph)

_lib.pgc_workspace_bytes.restype = _sz
_lib.pgc_workspace_bytes.argtypes = [_i64, _i64]
_lib.pgc_host_workspace_bytes.restype = _sz
_lib.pgc_host_workspace_bytes.argtypes = [_i64, _i64]
_lib.pgc_adg_order.restype = ctypes.c_int
_lib.pgc_adg_order.argtypes = [_GP, _u32, _u32, _vp, _i32p, _vp, _sz, _vp]
_lib.pgc_adg_order_mode.restype = ctypes.c_int
_lib.pgc_adg_order_mode.argtypes = [_GP, _u32, _u32, ctypes.c_int, _vp, _i32p, _vp, _sz, _vp]
_lib.pgc_jp_color.restype = ctypes.c_int
_lib.pgc_jp_color.argtypes = [_GP, _vp, _u64, _vp, _i32p, _vp, _sz, _vp]
_lib.pgc_color_jp_adg.restype = ctypes.c_int
_lib.pgc_color_jp_adg.argtypes = [_GP, _u32, _u32, _u64, _vp, _vp, _i32p, _i32p, _vp, _sz, _vp]
_lib.pgc_adg_m_order.restype = ctypes.c_int
_lib.pgc_adg_m_order.argtypes = [_GP, _vp, _i32p, _vp, _sz, _vp]
_lib.pgc_color_jp_adg_m.restype = ctypes.c_int
_lib.pgc_color_jp_adg_m.argtypes = [_GP, _u64, _vp, _vp, _i32p, _i32p, _vp, _sz, _vp]
_lib.pgc_color_jp_adg_o.restype = ctypes.c_int
_lib.pgc_color_jp_adg_o.argtypes = [_GP, _u32, _u32, _vp, _vp, _i32p, _i32p, _vp, _sz, _vp]
_lib.pgc_jp_baseline.restype = ctypes.c_int
_lib.pgc_jp_baseline.argtypes = [_GP, ctypes.c_int, _u64, _vp, _i32p, _vp, _sz, _vp]
_lib.pgc_color_dec_adg_itr.restype = ctypes.c_int
_lib.pgc_color_dec_adg_itr.argtypes = [_GP, _u32, _u32, _u64, _vp, _vp, _i32p, _i32p, _vp, _sz, _vp]
_lib.pgc_color_jp_adg_host.restype = ctypes.c_int
_lib.pgc_color_jp_adg_host.argtypes = [_i64, _i64, _vp, _vp, _u32, _u32, _u64, _vp, _vp, _i32p,
                                       _i32p, _vp, _sz, _vp]
_lib.pgc_check_graph.restype = ctypes.c_int
_lib.pgc_check_graph.argtypes = [_GP, _vp, _sz, _vp]
_lib.pgc_last_stats.restype = ctypes.c_int
_lib.pgc_last_stats.argtypes = [ctypes.POINTER(Stats)]
_lib.pgc_last_error.restype = ctypes.c_char_p
_lib.pgc_last_error.argtypes = []
_lib.pgc_set_tuning.restype = ctypes.c_int
_lib.pgc_set_tuning.argtypes = [ctypes.c_char_p, _i64]
_lib.pgc_version.restype = ctypes.c_int
_lib.pgc_version.argtypes = []
if hasattr(_lib, "pgc_debug_set_trace"):
    _lib.pgc_debug_set_trace.restype = ctypes.c_int
    _lib.pgc_debug_set_trace.argtypes = [_vp, _vp, _i64]


class PGCError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pgc error {code}: {msg}")
        self.code = code


def _check(rc: int):
    if rc != PGC_OK:
        raise PGCError(rc, _lib.pgc_last_error().decode(errors="replace"))


def _run(dev, fn, *args):
    """Call a library entry point with `dev` as the current CUDA device: the
    library takes the SM count, side streams and events from the current
    device, which must be the one the tensors and the stream live on."""
    with torch.cuda.device(dev):
        _check(fn(*args))


def lib():
    """The loaded ctypes library (for ABI tests)."""
    return _lib


def version() -> int:
    return _lib.pgc_version()


def workspace_bytes(n: int, nnz: int) -> int:
    return int(_lib.pgc_workspace_bytes(n, nnz))


def host_workspace_bytes(n: int, nnz: int) -> int:
    return int(_lib.pgc_host_workspace_bytes(n, nnz))


def set_tuning(key: str, value: int):
    _check(_lib.pgc_set_tuning(key.encode(), int(value)))


def debug_set_trace(t_grab=None, t_done=None):
    """Diagnostics (include/pgc_debug.h): record per-vertex JP grab/done
    %globaltimer stamps into two CUDA int64 tensors of n entries; None = off."""
    if t_grab is None:
        _check(_lib.pgc_debug_set_trace(None, None, 0))
    else:
        _check(_lib.pgc_debug_set_trace(t_grab.data_ptr(), t_done.data_ptr(), t_grab.numel()))


def last_stats() -> dict:
    s = Stats()
    _check(_lib.pgc_last_stats(ctypes.byref(s)))
    return {f: getattr(s, f) for f, _ in Stats._fields_}


_ws_cache: dict = {}


def _workspace(nbytes: int, device) -> torch.Tensor:
    key = (str(device),)
    t = _ws_cache.get(key)
    if t is None or t.numel() < nbytes:
        _ws_cache.pop(key, None)
        t = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_cache[key] = t
    return t


def release_workspace():
    _ws_cache.clear()


def _graph(row_offsets: torch.Tensor, col_indices: torch.Tensor) -> Graph:
    if not (row_offsets.is_cuda and col_indices.is_cuda):
        raise ValueError("row_offsets and col_indices must be CUDA tensors")
    if row_offsets.dtype != torch.int64 or col_indices.dtype != torch.int32:
        raise ValueError("row_offsets must be int64 and col_indices int32")
    if not (row_offsets.is_contiguous() and col_indices.is_contiguous()):
        raise ValueError("tensors must be contiguous")
    n = row_offsets.numel() - 1
    if n < 0:
        raise ValueError("row_offsets needs n+1 >= 1 entries")
    return Graph(n, col_indices.numel(), row_offsets.data_ptr(),
                 col_indices.data_ptr() if col_indices.numel() else None)


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _out(t, n, device, name):
    if t is None:
        return torch.empty(n, dtype=torch.int32, device=device)
    if t.dtype != torch.int32 or not t.is_cuda or t.numel() != n or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous CUDA int32 tensor with n entries")
    return t


UPDATE_MODES = {"push": 0, "pull": 1}   # enum pgc_update_mode


def adg_order(row_offsets, col_indices, eps_num: int, eps_den: int, *, update="push",
              round_out=None):
    """ADG ordering (Alg. 1) with the push or pull UPDATE.
    Returns (round int32[n] on device, T)."""
    g = _graph(row_offsets, col_indices)
    dev = row_offsets.device
    rnd = _out(round_out, g.n, dev, "round_out")
    nb = workspace_bytes(g.n, g.nnz)
    ws = _workspace(nb, dev)
    T = ctypes.c_int32(0)
    mode = UPDATE_MODES[update]
    _run(dev, _lib.pgc_adg_order_mode, ctypes.byref(g), eps_num, eps_den, mode,
                                   rnd.data_ptr() if g.n else None, ctypes.byref(T),
                                   ws.data_ptr(), ws.numel(), _stream(dev))
    return rnd, T.value


def jp_color(row_offsets, col_indices, round_key, seed: int, *, color_out=None):
    """JP coloring (Alg. 3) for priority <round_key, splitmix64(seed^v)>.  Returns (color, K)."""
    g = _graph(row_offsets, col_indices)
    dev = row_offsets.device
    if round_key.dtype != torch.int32 or not round_key.is_cuda or round_key.numel() != g.n:
        raise ValueError("round_key must be a CUDA int32 tensor with n entries")
    color = _out(color_out, g.n, dev, "color_out")
    ws = _workspace(workspace_bytes(g.n, g.nnz), dev)
    K = ctypes.c_int32(0)
    _run(dev, _lib.pgc_jp_color, ctypes.byref(g), round_key.contiguous().data_ptr() if g.n else None,
                             seed & 0xFFFFFFFFFFFFFFFF, color.data_ptr() if g.n else None,
                             ctypes.byref(K), ws.data_ptr(), ws.numel(), _stream(dev))
    return color, K.value


def color_jp_adg(row_offsets, col_indices, eps_num: int, eps_den: int, seed: int, *,
                 round_out=None, color_out=None):
    """JP-ADG (the whole hot path).  Returns (round, color, T, K)."""
    g = _graph(row_offsets, col_indices)
    dev = row_offsets.device
    rnd = _out(round_out, g.n, dev, "round_out")
    color = _out(color_out, g.n, dev, "color_out")
    ws = _workspace(workspace_bytes(g.n, g.nnz), dev)
    T, K = ctypes.c_int32(0), ctypes.c_int32(0)
    _run(dev, _lib.pgc_color_jp_adg, ctypes.byref(g), eps_num, eps_den, seed & 0xFFFFFFFFFFFFFFFF,
                                 rnd.data_ptr() if g.n else None, color.data_ptr() if g.n else None,
                                 ctypes.byref(T), ctypes.byref(K), ws.data_ptr(), ws.numel(),
                                 _stream(dev))
    return rnd, color, T.value, K.value


def adg_m_order(row_offsets, col_indices, *, round_out=None):
    """ADG-M ordering (median rule).  Returns (round int32[n], T)."""
    g = _graph(row_offsets, col_indices)
    dev = row_offsets.device
    rnd = _out(round_out, g.n, dev, "round_out")
    ws = _workspace(workspace_bytes(g.n, g.nnz), dev)
    T = ctypes.c_int32(0)
    _run(dev, _lib.pgc_adg_m_order, ctypes.byref(g), rnd.data_ptr() if g.n else None, ctypes.byref(T),
                                ws.data_ptr(), ws.numel(), _stream(dev))
    return rnd, T.value


def color_jp_adg_m(row_offsets, col_indices, seed: int, *, round_out=None, color_out=None):
    """JP-ADG-M.  Returns (round, color, T, K)."""
    g = _graph(row_offsets, col_indices)
    dev = row_offsets.device
    rnd = _out(round_out, g.n, dev, "round_out")
    color = _out(color_out, g.n, dev, "color_out")
    ws = _workspace(workspace_bytes(g.n, g.nnz), dev)
    T, K = ctypes.c_int32(0), ctypes.c_int32(0)
    _run(dev, _lib.pgc_color_jp_adg_m, ctypes.byref(g), seed & 0xFFFFFFFFFFFFFFFF,
                                   rnd.data_ptr() if g.n else None, color.data_ptr() if g.n else None,
                                   ctypes.byref(T), ctypes.byref(K), ws.data_ptr(), ws.numel(),
                                   _stream(dev))
    return rnd, color, T.value, K.value


def color_jp_adg_o(row_offsets, col_indices, eps_num: int, eps_den: int, *, round_out=None,
                   color_out=None):
    """JP-ADG-O (ADG-O's total order).  Returns (round, color, T, K)."""
    g = _graph(row_offsets, col_indices)
    dev = row_offsets.device
    rnd = _out(round_out, g.n, dev, "round_out")
    color = _out(color_out, g.n, dev, "color_out")
    ws = _workspace(workspace_bytes(g.n, g.nnz), dev)
    T, K = ctypes.c_int32(0), ctypes.c_int32(0)
    _run(dev, _lib.pgc_color_jp_adg_o, ctypes.byref(g), eps_num, eps_den,
                                   rnd.data_ptr() if g.n else None, color.data_ptr() if g.n else None,
                                   ctypes.byref(T), ctypes.byref(K), ws.data_ptr(), ws.numel(),
                                   _stream(dev))
    return rnd, color, T.value, K.value


JP_KINDS = {"jp-r": 0, "jp-ff": 1, "jp-lf": 2, "jp-llf": 3}


def jp_baseline(row_offsets, col_indices, kind: str, seed: int, *, color_out=None):
    """JP-R / JP-FF / JP-LF / JP-LLF.  Returns (color, K)."""
    g = _graph(row_offsets, col_indices)
    dev = row_offsets.device
    color = _out(color_out, g.n, dev, "color_out")
    ws = _workspace(workspace_bytes(g.n, g.nnz), dev)
    K = ctypes.c_int32(0)
    _run(dev, _lib.pgc_jp_baseline, ctypes.byref(g), JP_KINDS[kind], seed & 0xFFFFFFFFFFFFFFFF,
                                color.data_ptr() if g.n else None, ctypes.byref(K), ws.data_ptr(),
                                ws.numel(), _stream(dev))
    return color, K.value


def color_dec_adg_itr(row_offsets, col_indices, eps_num: int, eps_den: int, seed: int, *,
                      round_out=None, color_out=None):
    """DEC-ADG-ITR.  Returns (round, color, T, K)."""
    g = _graph(row_offsets, col_indices)
    dev = row_offsets.device
    rnd = _out(round_out, g.n, dev, "round_out")
    color = _out(color_out, g.n, dev, "color_out")
    ws = _workspace(workspace_bytes(g.n, g.nnz), dev)
    T, K = ctypes.c_int32(0), ctypes.c_int32(0)
    _run(dev, _lib.pgc_color_dec_adg_itr, ctypes.byref(g), eps_num, eps_den, seed & 0xFFFFFFFFFFFFFFFF,
                                      rnd.data_ptr() if g.n else None,
                                      color.data_ptr() if g.n else None, ctypes.byref(T),
                                      ctypes.byref(K), ws.data_ptr(), ws.numel(), _stream(dev))
    return rnd, color, T.value, K.value


def color_jp_adg_host(row_offsets, col_indices, eps_num: int, eps_den: int, seed: int,
                      round_out, color_out, device=None):
    """JP-ADG from HOST (ideally pinned) CPU tensors; outputs written to host tensors.
    Host<->device copies happen inside the call.  Returns (T, K)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    for t, dt in ((row_offsets, torch.int64), (col_indices, torch.int32), (round_out, torch.int32),
                  (color_out, torch.int32)):
        if t.is_cuda or t.dtype != dt or not t.is_contiguous():
            raise ValueError("host tensors must be contiguous CPU tensors of the documented dtypes")
    n, nnz = row_offsets.numel() - 1, col_indices.numel()
    ws = _workspace(host_workspace_bytes(n, nnz), dev)
    T, K = ctypes.c_int32(0), ctypes.c_int32(0)
    _run(dev, _lib.pgc_color_jp_adg_host, n, nnz, row_offsets.data_ptr(),
                                      col_indices.data_ptr() if nnz else None, eps_num, eps_den,
                                      seed & 0xFFFFFFFFFFFFFFFF,
                                      round_out.data_ptr() if n else None,
                                      color_out.data_ptr() if n else None,
                                      ctypes.byref(T), ctypes.byref(K), ws.data_ptr(), ws.numel(),
                                      _stream(dev))
    return T.value, K.value


def check_graph(row_offsets, col_indices):
    """Validate CSR invariants on the device; raises PGCError(PGC_EINVAL) on a violation."""
    g = _graph(row_offsets, col_indices)
    dev = row_offsets.device
    ws = _workspace(workspace_bytes(g.n, g.nnz), dev)
    _run(dev, _lib.pgc_check_graph, ctypes.byref(g), ws.data_ptr(), ws.numel(), _stream(dev))
