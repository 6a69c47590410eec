#!/usr/bin/env python
"""Top warp-stall SASS instructions of one kernel launch in an ncu report.
  python tools/ncu_hot.py report.ncu-rep <launch-index> [N]"""
import csv
import subprocess
import sys


def main():
    rep, k = sys.argv[1], int(sys.argv[2])
    N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(k),
                          "--launch-count", "1", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
    h = rows[hi]
    ai, si, wi = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[hi + 1:]:
        try:
            data.append((float(r[wi] or 0), r[ai], r[si]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    order = {d[1]: i for i, d in enumerate(data)}
    print(rows[0][1][:120] if len(rows[0]) > 1 else "")
    for w, a, s in sorted(data, key=lambda d: -d[0])[:N]:
        print(f"{100 * w / tot:5.1f}%  #{order[a]:4d} {a}  {s[:100]}")


if __name__ == "__main__":
    main()
