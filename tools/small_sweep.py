#!/usr/bin/env python
"""Time the one-kernel small path (csrc/small.cu) against the multi-kernel
path on the small configs, over a few tuning values (CUDA events, warm)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_2008_11321_b200 as pgc  # noqa: E402


def timed(off, col, num, den, reps=20):
    for _ in range(3):
        pgc.color_jp_adg(off, col, num, den, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pgc.color_jp_adg(off, col, num, den, 1)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name in (sys.argv[1:] or ["er", "grid", "rmat20"]):
    g = gg.config_graph(name)
    num, den = gg.CONFIGS[name][1][0]
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda()
    pgc.set_tuning("small_max_arcs", 0)
    print(name, "multi-kernel", "%.3f ms" % timed(off, col, num, den), flush=True)
    pgc.set_tuning("small_max_arcs", 1 << 40)
    pgc.set_tuning("small_max_avg", 1 << 30)
    for bps in (1, 2, 0):
        pgc.set_tuning("small_blocks_per_sm", bps)
        t = timed(off, col, num, den)
        st = pgc.last_stats()
        print(name, "small bps=%d" % bps, "%.3f ms" % t, "T", st["rounds"], "small", st["small_path"], flush=True)
    pgc.set_tuning("small_blocks_per_sm", 0)
    for df in (0, 1):
        pgc.set_tuning("tiny_dataflow", df)
        t = timed(off, col, num, den)
        st = pgc.last_stats()
        print(name, "tiny_dataflow=%d" % df, "%.3f ms" % t, "small", st["small_path"], flush=True)
    pgc.set_tuning("tiny_dataflow", 1)
    pgc.set_tuning("small_max_arcs", 1 << 24)
    pgc.set_tuning("small_max_avg", 20)
