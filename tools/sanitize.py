#!/usr/bin/env python
"""Checked runs: every C-ABI entry point once on one
graph, each result checked against the oracle, with output buffers poisoned
before each call.  compute-sanitizer is closed on the GPU pool, so this runs
on the checked library (tools/micro/build_checked.sh: device bounds asserts,
workspace canaries, a poisoned workspace per call):

  PGC_LIB=tools/micro/libpgc_checked.so python tools/sanitize.py er
  CUDA_LAUNCH_BLOCKING=1 PGC_LIB=... python tools/sanitize.py rmat16 --serial

Graphs: er (config 1), grid (config 3), rmat20 (config 2), or rmatS (scale S).
--entries restricts the entry points (comma list).  The JP watchdog is raised
to an hour: instrumented kernels run orders of magnitude slower.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle as O  # noqa: E402
import paper_2008_11321_b200 as pgc  # noqa: E402

ALL = ["jp_adg", "jp_adg_small", "jp_adg_multi", "adg_push", "adg_pull", "jp_color", "jp_adg_o",
       "jp_adg_m", "jp_r", "dec_adg_itr", "host"]


def graph(name):
    if name in gg.CONFIGS:
        return gg.config_graph(name), gg.CONFIGS[name][1][0]
    if name.startswith("rmat"):
        return gg.rmat(int(name[4:]), 16, seed=1), (1, 10)
    raise SystemExit(f"unknown graph {name}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("graph")
    ap.add_argument("--entries", default=",".join(ALL))
    ap.add_argument("--serial", action="store_true", help="one-stream JP schedule")
    a = ap.parse_args()
    pgc.set_tuning("jp_watchdog_ms", 3600000)
    if a.serial:
        pgc.set_tuning("jp_split_overlap", 0)
    g, (num, den) = graph(a.graph)
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda()
    r_or, _ = O.adg(g, num, den)
    c_or, K_or = O.jp(g, r_or, 1)
    ok = True

    def check(name, cond):
        nonlocal ok
        print(f"{name}: {'ok' if cond else 'MISMATCH'}", flush=True)
        ok &= bool(cond)

    POISON = -0x5a5a5a5b

    def outs():
        return (torch.full((g.n,), POISON, dtype=torch.int32, device="cuda"),
                torch.full((g.n,), POISON, dtype=torch.int32, device="cuda"))

    for e in a.entries.split(","):
        t0 = time.time()
        ro, co = outs()
        if e in ("jp_adg", "jp_adg_small", "jp_adg_multi"):
            # default heuristic, then the one-kernel path and the multi-kernel path forced
            if e == "jp_adg_small":
                pgc.set_tuning("small_max_arcs", 1 << 40)
                pgc.set_tuning("small_max_avg", 1 << 30)
            elif e == "jp_adg_multi":
                pgc.set_tuning("small_max_arcs", 0)
            r, c, T, K = pgc.color_jp_adg(off, col, num, den, 1, round_out=ro, color_out=co)
            path = pgc.last_stats()["small_path"]
            pgc.set_tuning("small_max_arcs", 1 << 24)
            pgc.set_tuning("small_max_avg", 20)
            check(f"{e} (small_path={path})",
                  np.array_equal(r.cpu().numpy(), r_or) and np.array_equal(c.cpu().numpy(), c_or))
        elif e in ("adg_push", "adg_pull"):
            r, T = pgc.adg_order(off, col, num, den, update=e[4:], round_out=ro)
            check(e, np.array_equal(r.cpu().numpy(), r_or))
        elif e == "jp_color":
            c, K = pgc.jp_color(off, col, torch.from_numpy(r_or).cuda(), 1, color_out=co)
            check(e, np.array_equal(c.cpu().numpy(), c_or))
        elif e == "jp_adg_o":
            r, c, T, K = pgc.color_jp_adg_o(off, col, num, den, round_out=ro, color_out=co)
            r_o, rho, _, _, _ = O.adg_o(g, num, den)
            c_o, _ = O.jp_rho(g, rho)
            check(e, np.array_equal(r.cpu().numpy(), r_o) and np.array_equal(c.cpu().numpy(), c_o))
        elif e == "jp_adg_m":
            r, c, T, K = pgc.color_jp_adg_m(off, col, 1, round_out=ro, color_out=co)
            r_m, _ = O.adg_m(g)
            c_m, _ = O.jp(g, r_m, 1)
            check(e, np.array_equal(r.cpu().numpy(), r_m) and np.array_equal(c.cpu().numpy(), c_m))
        elif e == "jp_r":
            c, K = pgc.jp_baseline(off, col, "jp-r", 1, color_out=co)
            c_r, _ = O.jp(g, np.zeros(g.n, np.int32), 1)
            check(e, np.array_equal(c.cpu().numpy(), c_r))
        elif e == "dec_adg_itr":
            r, c, T, K = pgc.color_dec_adg_itr(off, col, num, den, 1, round_out=ro, color_out=co)
            c_d, _, _ = O.dec_adg_itr(g, r_or, 1)
            check(e, np.array_equal(c.cpu().numpy(), c_d))
        elif e == "host":
            h_r = torch.full((g.n,), POISON, dtype=torch.int32).pin_memory()
            h_c = torch.full((g.n,), POISON, dtype=torch.int32).pin_memory()
            pgc.color_jp_adg_host(torch.from_numpy(g.off), torch.from_numpy(g.col), num, den, 1, h_r, h_c)
            check(e, np.array_equal(h_r.numpy(), r_or) and np.array_equal(h_c.numpy(), c_or))
        torch.cuda.synchronize()
        print(f"  {e} {time.time() - t0:.1f} s", flush=True)
    print(f"lib: {pgc.SO_PATH}")
    print("ALL OK" if ok else "FAILED")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
