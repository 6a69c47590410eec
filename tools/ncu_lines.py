#!/usr/bin/env python
"""Per-source-line instruction and stall-sample shares of one launch in an ncu report.
  python tools/ncu_lines.py report.ncu-rep [launch-index] [N]"""
import collections
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(k),
                          "--launch-count", "1", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
    h = rows[hi]
    ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    fname = ""
    line = None
    agg, st, src = collections.Counter(), collections.Counter(), {}
    for r in rows[hi + 1:]:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) <= ie:
            continue
        if r[0].isdigit():
            line = (fname, int(r[0]))
            src[line] = r[1]
        try:
            x, y = float(r[ie] or 0), float(r[ws] or 0)
        except ValueError:
            continue
        if line is not None:
            agg[line] += x
            st[line] += y
    tot, tots = sum(agg.values()) or 1, sum(st.values()) or 1
    for l, x in sorted(st.items(), key=lambda t: -t[1])[:N]:
        print(f"{100 * st[l] / tots:5.1f}% stall {100 * agg[l] / tot:5.1f}% inst  {l[0]}:{l[1]}: {src.get(l, '')[:90]}")


if __name__ == "__main__":
    main()
