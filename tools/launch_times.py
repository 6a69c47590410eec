#!/usr/bin/env python
"""Per-launch kernel times for tuning variants (run under ncu, see --help).

  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_update --csv \
      --log-file out.csv python tools/launch_times.py --config rmat24 filter_ratio=0 filter_ratio=6
Each variant runs twice (warm, then the profiled pass); parse with --parse out.csv.
"""
import argparse
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parse(path, nvar):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ks = [(r[ki].split("(")[0], float(r[vi].replace(",", "")) / 1e3) for r in rows[1:]]
    per = len(ks) // (2 * nvar)
    for j in range(nvar):
        seg = ks[(2 * j + 1) * per:(2 * j + 2) * per]
        print(f"variant {j}: total {sum(t for _, t in seg):.3f} us->ms")
        for name, t in seg:
            print(f"   {name:40s} {t:8.1f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="rmat24")
    ap.add_argument("--parse", default=None)
    ap.add_argument("variants", nargs="*")
    a = ap.parse_args()
    if a.parse:
        return parse(a.parse, max(1, len(a.variants)))
    import torch
    import graphgen as gg
    import paper_2008_11321_b200 as pgc
    path = f"/tmp/pgc_graph_{a.config}.npz"
    if os.path.exists(path):
        import numpy as np
        z = np.load(path)
        g = gg.Graph(len(z["off"]) - 1, z["off"], z["col"], a.config)
    else:
        import numpy as np
        g = gg.config_graph(a.config)
        np.savez(path, off=g.off, col=g.col)
    num, den = gg.CONFIGS[a.config][1][0]
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda()
    for var in a.variants or [""]:
        for kv in filter(None, var.split(",")):
            k, v = kv.split("=")
            pgc.set_tuning(k, int(v))
        for _ in range(2):
            pgc.color_jp_adg(off, col, num, den, 1)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
