#!/usr/bin/env python
"""JP-ADG step time with and without the core_div cap on mid-size R-MAT graphs
(scales 16-19: between the one-kernel path's graphs and BASELINE's R-MAT 20).
  python tools/core_div_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import graphgen as gg
import paper_2008_11321_b200 as pgc

for scale in (16, 17, 18, 19):
    g = gg.rmat(scale, 16, seed=1)
    off, col = torch.from_numpy(g.off).cuda(), torch.from_numpy(g.col).cuda()
    for div in (0, 32, 0, 32):
        pgc.set_tuning("core_div", div)
        for _ in range(3):
            pgc.color_jp_adg(off, col, 1, 10, 1)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            pgc.color_jp_adg(off, col, 1, 10, 1)
        b.record()
        torch.cuda.synchronize()
        st = pgc.last_stats()
        print(f"rmat{scale} core_div={div}: {a.elapsed_time(b) / 20:.3f} ms/step, core {st['core_vertices']} "
              f"vertices, small_path {st.get('small_path')}", flush=True)
pgc.set_tuning("core_div", 32)
