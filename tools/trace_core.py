#!/usr/bin/env python
"""Dump per-vertex JP trace stamps (grab/done, %globaltimer ns) with priority
position, round, |pred| and JP level for the first `--keep` priority positions
(the core and what follows) to an .npz for offline analysis.
  python tools/trace_core.py --config rmat24 --out gpurun_out/core_trace.npz
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle as O  # noqa: E402
from _refcheck import _hash_np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="rmat24")
    ap.add_argument("--eps", default=None)
    ap.add_argument("--keep", type=int, default=400000)
    ap.add_argument("--out", required=True)
    ap.add_argument("--tune", nargs="*", default=[])
    a = ap.parse_args()
    import paper_2008_11321_b200 as pgc
    for kv in a.tune:
        k, val = kv.split("=")
        pgc.set_tuning(k, int(val))
    g = gg.config_graph(a.config)
    num, den = map(int, a.eps.split("/")) if a.eps else gg.CONFIGS[a.config][1][0]
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda()
    tg = torch.zeros(g.n, dtype=torch.int64, device="cuda")
    td = torch.zeros(g.n, dtype=torch.int64, device="cuda")
    pgc.color_jp_adg(off, col, num, den, 1)
    pgc.set_tuning("timing", 1)
    pgc.debug_set_trace(tg, td)
    rnd, color, T, K = pgc.color_jp_adg(off, col, num, den, 1)
    st = pgc.last_stats()
    pgc.debug_set_trace(None, None)
    r = rnd.cpu().numpy()
    h = _hash_np(g.n, 1)
    key = np.lexsort((h, r))[::-1][:a.keep]       # priority order prefix
    _, _, lvl, J = O.jp(g, r, 1, levels=True)
    deg = np.diff(g.off)
    # |pred| per kept vertex
    npred = np.zeros(len(key), dtype=np.int64)
    for i, v in enumerate(key):
        nb = g.col[g.off[v]:g.off[v + 1]]
        npred[i] = int(((r[nb] > r[v]) | ((r[nb] == r[v]) & (h[nb] > h[v]))).sum())
    tgc, tdc = tg.cpu().numpy(), td.cpu().numpy()
    np.savez(a.out, v=key, tg=tgc[key], td=tdc[key], level=lvl[key], round=r[key], npred=npred,
             deg=deg[key], core_n=st["core_vertices"], core_ctas=st["core_ctas"],
             t_core_ms=st["t_core_ms"], t_jp_ms=st["t_jp_ms"], J=J, T=T, K=K)
    print("saved", a.out, st["core_vertices"], st["core_ctas"], st["t_core_ms"], st["t_jp_ms"])


if __name__ == "__main__":
    main()
