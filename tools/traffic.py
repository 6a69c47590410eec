#!/usr/bin/env python
"""DRAM traffic of one step's UPDATE launches per workload (the roofline's
`traffic` in bench.py), measured with ncu on the GPU box.

  # on the box: a plain run first, then the same command under ncu
  python tools/traffic.py run --config rmat24 --eps 1/10 &&
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:k_update --csv --log-file gpurun_out/t.csv \
      python tools/traffic.py run --config rmat24 --eps 1/10
  # here: merge into profiles/traffic.json (keyed like bench.py's config.workload)
  python tools/traffic.py parse gpurun_out/t.csv --workload rmat24-eps1/10 --source <path>

`run` makes two JP-ADG calls (the first warms up); `parse` sums the second
call's k_update* launches (half of the captured launches).  Workloads on the
one-kernel small-graph path (csrc/small.cu) have no UPDATE launch: capture
`-k regex:k_small` and parse with `--kernel k_small_jp_adg --workload
<workload>-small` (the whole path's DRAM bytes, bench.py's `traffic` there).
"""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(a):
    import numpy as np
    import torch
    import graphgen as gg
    import paper_2008_11321_b200 as pgc
    path = f"/tmp/pgc_graph_{a.config}.npz"
    if os.path.exists(path):
        z = np.load(path)
        g = gg.Graph(len(z["off"]) - 1, z["off"], z["col"], a.config)
    else:
        g = gg.config_graph(a.config)
        np.savez(path, off=g.off, col=g.col)
    num, den = (int(x) for x in a.eps.split("/")) if a.eps else gg.CONFIGS[a.config][1][0]
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda()
    for _ in range(2):
        pgc.color_jp_adg(off, col, num, den, 1)
    torch.cuda.synchronize()


def parse(a):
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
    h = rows[0]
    ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    kp = a.kernel
    ids = sorted({int(r[ii]) for r in rows[1:] if r[ki].startswith("void " + kp) or
                  r[ki].startswith(kp)})
    second = set(ids[len(ids) // 2:])   # the second (profiled) call's launches
    # ncu reports bytes with unit prefixes in some versions: the csv unit column says which
    ui = h.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = sum(float(r[vi].replace(",", "")) * scale.get(r[ui], 1) for r in rows[1:]
             if int(r[ii]) in second and r[ni] == "dram__bytes_read.sum")
    wr = sum(float(r[vi].replace(",", "")) * scale.get(r[ui], 1) for r in rows[1:]
             if int(r[ii]) in second and r[ni] == "dram__bytes_write.sum")
    p = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d[a.workload] = {"update_dram_bytes_per_step": rd + wr, "read": rd, "write": wr,
                     "launches": len(second), "source": a.source or a.csv}
    json.dump(d, open(p, "w"), indent=1, sort_keys=True)
    print(a.workload, rd + wr, len(second))


def main():
    ap = argparse.ArgumentParser()
    sp = ap.add_subparsers(dest="cmd", required=True)
    r = sp.add_parser("run")
    r.add_argument("--config", default="rmat24")
    r.add_argument("--eps", default=None)
    q = sp.add_parser("parse")
    q.add_argument("csv")
    q.add_argument("--workload", required=True)
    q.add_argument("--source", default=None)
    q.add_argument("--kernel", default="k_update",
                   help="kernel name prefix (k_small_jp_adg for the one-kernel path; "
                        "its workload key gets the suffix -small)")
    a = ap.parse_args()
    return run(a) if a.cmd == "run" else parse(a)


if __name__ == "__main__":
    main()
