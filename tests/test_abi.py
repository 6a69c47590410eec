"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/pgc.h declares, and rejects bad arguments before touching CUDA."""
import ctypes
import os
import re

import pytest

import paper_2008_11321_b200 as pgc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = "".join(open(os.path.join(ROOT, "include", f)).read()
                  for f in sorted(os.listdir(os.path.join(ROOT, "include"))) if f.endswith(".h"))
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pgc_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_contract():
    names = header_functions()
    for required in ("pgc_adg_order", "pgc_jp_color", "pgc_color_jp_adg", "pgc_workspace_bytes",
                     "pgc_last_error", "pgc_last_stats"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = pgc.lib()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert sorted(pgc.EXPORTS) == header_functions()


def test_exports_are_extern_c():
    out = os.popen(f"nm -D --defined-only {pgc.SO_PATH}").read()
    for name in header_functions():
        assert re.search(rf"\bT {name}$", out, flags=re.M), name


def test_version_and_workspace_sizes():
    hdr = open(os.path.join(ROOT, "include", "pgc.h")).read()
    declared = int(re.search(r"#define PGC_VERSION (\d+)", hdr).group(1))
    assert pgc.version() == declared
    assert pgc.workspace_bytes(0, 0) > 0
    a = pgc.workspace_bytes(1000, 10000)
    b = pgc.workspace_bytes(2000, 10000)
    c = pgc.workspace_bytes(1000, 20000)
    assert b > a and c > a
    assert a % 256 == 0
    assert pgc.workspace_bytes(-1, 0) == 0 and pgc.workspace_bytes(1 << 29, 0) == 0
    assert pgc.workspace_bytes(10, -1) == 0
    assert pgc.host_workspace_bytes(1000, 10000) > a


def test_tuning_validation():
    pgc.set_tuning("rounds_per_sync", 4)
    pgc.set_tuning("rounds_per_sync", 8)
    for key, val in (("nope", 1), ("heavy_degree", 3), ("block_threads", 100), ("timing", 2)):
        with pytest.raises(pgc.PGCError) as e:
            pgc.set_tuning(key, val)
        assert e.value.code == pgc.PGC_EINVAL


def _call_adg(g, num=1, den=10, ws=None, wsb=0):
    T = ctypes.c_int32(-7)
    rc = pgc.lib().pgc_adg_order(ctypes.byref(g) if g is not None else None, num, den,
                                 ctypes.c_void_p(0x1000), ctypes.byref(T), ws, wsb, None)
    return rc, T.value


def test_argument_errors_without_gpu():
    lib = pgc.lib()
    rc, _ = _call_adg(None)
    assert rc == pgc.PGC_EINVAL and b"NULL" in lib.pgc_last_error()
    g = pgc.Graph(-1, 0, 0x1000, 0x2000)
    assert _call_adg(g)[0] == pgc.PGC_EINVAL
    g = pgc.Graph(1 << 29, 0, 0x1000, 0x2000)
    assert _call_adg(g)[0] == pgc.PGC_EINVAL
    g = pgc.Graph(10, 20, None, 0x2000)
    assert _call_adg(g)[0] == pgc.PGC_EINVAL
    g = pgc.Graph(10, 20, 0x1000, None)
    assert _call_adg(g)[0] == pgc.PGC_EINVAL
    g = pgc.Graph(10, 20, 0x1000, 0x2000)
    assert _call_adg(g, num=0)[0] == pgc.PGC_EINVAL
    assert _call_adg(g, den=0)[0] == pgc.PGC_EINVAL
    assert _call_adg(g, ws=None, wsb=1 << 30)[0] == pgc.PGC_EWORKSPACE
    assert _call_adg(g, ws=0x1001, wsb=1 << 30)[0] == pgc.PGC_EWORKSPACE       # misaligned
    assert _call_adg(g, ws=0x10000, wsb=16)[0] == pgc.PGC_EWORKSPACE          # too small
    assert b"too small" in lib.pgc_last_error()
    K = ctypes.c_int32(0)
    rc = lib.pgc_jp_color(ctypes.byref(g), None, 1, ctypes.c_void_p(0x1000), ctypes.byref(K),
                          ctypes.c_void_p(0x10000), 1 << 30, None)
    assert rc == pgc.PGC_EINVAL
    T = ctypes.c_int32(0)
    rc = lib.pgc_color_jp_adg(ctypes.byref(g), 1, 10, 1, ctypes.c_void_p(0x1000), None,
                              ctypes.byref(T), ctypes.byref(K), ctypes.c_void_p(0x10000), 1 << 30, None)
    assert rc == pgc.PGC_EINVAL
    assert lib.pgc_last_stats(None) == pgc.PGC_EINVAL
    for mode in (-1, 2):   # enum pgc_update_mode has PUSH = 0 and PULL = 1 only
        rc = lib.pgc_adg_order_mode(ctypes.byref(g), 1, 10, mode, ctypes.c_void_p(0x1000),
                                    ctypes.byref(T), ctypes.c_void_p(0x10000), 1 << 30, None)
        assert rc == pgc.PGC_EINVAL and b"update_mode" in lib.pgc_last_error()


def test_product_path_does_not_import_oracle():
    import subprocess, sys
    code = ("import sys, paper_2008_11321_b200; "
            "assert 'oracle' not in sys.modules, 'product imported the oracle'")
    subprocess.check_call([sys.executable, "-c", code], cwd=ROOT)
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2008_11321_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "oracle.h" not in src and "orc_" not in src, f
