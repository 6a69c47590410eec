#!/usr/bin/env python
"""Run the one-kernel small-graph path (csrc/small.cu) on a ladder of graphs,
each in a fresh process (a trap kills the context), and report the first
failure (use with PGC_LIB=tools/micro/libpgc_checked.so for bounds checks)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = sys.argv[1:] or ["er(300,1200,1)", "er(2000,8000,1)", "er(16384,131072,1)",
                         "rmat(10,8,seed=1)", "config_graph('er')", "config_graph('grid')"]
CODE = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import graphgen as gg, oracle as O, paper_2008_11321_b200 as pgc
pgc.set_tuning('small_max_arcs', 1 << 40); pgc.set_tuning('small_max_avg', 1 << 30)
g = gg.%s
off = torch.from_numpy(g.off).cuda(); col = torch.from_numpy(g.col).cuda()
r, c, T, K = pgc.color_jp_adg(off, col, 1, 10, 1)
torch.cuda.synchronize()
st = pgc.last_stats()
r_or, so = O.adg(g, 1, 10); c_or, K_or = O.jp(g, r_or, 1)
print('n', g.n, 'small', st['small_path'], 'T', T, so['T'], 'K', K, K_or,
      'round_ok', np.array_equal(r.cpu().numpy(), r_or), 'color_ok', np.array_equal(c.cpu().numpy(), c_or))
"""
for case in CASES:
    out = subprocess.run([sys.executable, "-c", CODE % (ROOT, case)], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    print(case, "rc", out.returncode, out.stdout.strip()[-400:], out.stderr.strip()[-1500:], flush=True)
