#!/usr/bin/env python
"""Tuning sweep on one config: per-group device times for each knob setting.

  python tools/sweep.py --config rmat24 --reps 3 hw=1,2,4 ctas=0,4,16
Results never depend on the knobs (checked here against the first setting).
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402

KEYS = {"hw": "jp_heavy_warps", "hsleep": "jp_heavy_sleep_max", "lsleep": "jp_light_sleep_max", "chunk": "chunk_arcs", "heavy_deg": "heavy_degree",
        "rps": "rounds_per_sync", "core": "core_max", "ctas": "core_ctas", "avg": "core_min_avg",
        "apc": "core_arcs_per_cta", "spin": "core_spin_ns", "near": "core_near", "pass": "core_pass_ns",
        "tail": "core_tail_ns", "hb": "jp_heavy_batch", "t2": "core_tier2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="rmat24")
    ap.add_argument("--eps", default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("knobs", nargs="*")
    a = ap.parse_args()
    import paper_2008_11321_b200 as pgc
    from bench import load_graph  # /tmp-cached generator output
    g = load_graph(a.config)
    num, den = map(int, a.eps.split("/")) if a.eps else gg.CONFIGS[a.config][1][0]
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda()
    grid = []
    for kv in a.knobs:
        k, vs = kv.split("=")
        grid.append([(KEYS.get(k, k), int(v)) for v in vs.split(",")])
    ref = None
    pgc.set_tuning("timing", 1)
    for combo in itertools.product(*grid) if grid else [()]:
        for k, v in combo:
            pgc.set_tuning(k, v)
        pgc.color_jp_adg(off, col, num, den, 1)  # warm
        rows = []
        for _ in range(a.reps):
            r, c, T, K = pgc.color_jp_adg(off, col, num, den, 1)
            rows.append(pgc.last_stats())
        out = (r.cpu().numpy(), c.cpu().numpy())
        if ref is None:
            ref = out
        same = bool(np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1]))
        med = {k: float(np.median([x[k] for x in rows])) for k in rows[0] if k.startswith("t_")}
        med["core_vertices"] = rows[-1]["core_vertices"]
        med["core_ctas"] = rows[-1]["core_ctas"]
        print(json.dumps({"config": a.config, "knobs": dict(combo), "same": same,
                          "edges_per_s": g.m / (med["t_total_ms"] * 1e-3), **med}), flush=True)


if __name__ == "__main__":
    main()
