#!/usr/bin/env python
"""JP dependency-chain latency probe: on K_n every vertex depends on all
higher-priority ones, so JP is a chain of n hops; t / n is the per-hop cost.
  python tools/chain_bench.py --n 1000 core_ctas=1,16 core_spin_ns=0,64
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import graphgen as gg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("knobs", nargs="*")
    a = ap.parse_args()
    import paper_2008_11321_b200 as pgc
    n = a.n
    g = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda()
    pgc.set_tuning("core_min_avg", 0)
    pgc.set_tuning("core_min_n", 1)
    pgc.set_tuning("timing", 1)
    grid = [[(k, int(v)) for v in vs.split(",")] for k, vs in (kv.split("=") for kv in a.knobs)]
    for combo in itertools.product(*grid):
        for k, v in combo:
            pgc.set_tuning(k, v)
        pgc.color_jp_adg(off, col, 1, 10, 1)
        ts = []
        for _ in range(a.reps):
            _, _, T, K = pgc.color_jp_adg(off, col, 1, 10, 1)
            st = pgc.last_stats()
            ts.append((st["t_core_ms"], st["t_jp_ms"]))
        core = min(t[0] for t in ts)
        bulk = min(t[1] for t in ts)
        print(json.dumps({"n": n, "knobs": dict(combo), "K": K, "core_ms": core, "bulk_ms": bulk,
                          "ns_per_hop": 1e6 * (core + bulk) / n,
                          "core_vertices": st["core_vertices"], "ctas": st["core_ctas"]}),
              flush=True)


if __name__ == "__main__":
    main()
