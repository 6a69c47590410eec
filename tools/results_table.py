#!/usr/bin/env python
"""BASELINE.md §4 results table from a directory of bench.py lines
(bench_<config>_<eps>.json, tools/r2_profile.sh stage `bench`) and the
per-workload UPDATE DRAM traffic (profiles/traffic.json).

  python tools/results_table.py profiles/r2_final
"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORDER = ["er-eps1/10", "rmat20-eps1/100", "rmat20-eps1/10", "rmat20-eps1/2", "grid-eps1/10",
         "rmat24-eps1/10", "cl-eps1/100", "cl-eps1/2"]
NAMES = {"er": "ER 16K/131K", "rmat20": "R-MAT 20", "grid": "Road-like 2048²", "rmat24": "**R-MAT 24**",
         "cl": "Chung-Lu 2²³"}


def main():
    src = sys.argv[1]
    lines = {}
    for f in glob.glob(os.path.join(src, "bench_*.json")):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception:
            continue
        lines[d["config"]["workload"]] = d
    tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    out = ["| Config | n | m | ε | T | J | K | d | GPU ms/step (median) | GPU edges/s | path % of 8 TB/s | "
           "path % of measured HBM | UPDATE % of measured HBM | UPDATE ncu DRAM GB/s | oracle s (1 core) | "
           "oracle edges/s | parity |",
           "|" + "---|" * 17]
    for w in ORDER:
        d = lines.get(w)
        if not d:
            continue
        c, rf = d["config"], d["roofline"]
        t = d["timing"]["median_ms"]
        cb = d.get("cpu_baseline", {})
        om = cb.get("oracle_ms", {})
        osec = (om.get("adg", 0) + om.get("jp", 0)) / 1e3 if om else None
        small = bool(d.get("small_path"))
        e = tr.get(w + "-small") if small else tr.get(w)
        dram = e["update_dram_bytes_per_step"] / (rf["ms_per_launch"] * 1e-3) / 1e9 if e else None
        par = d.get("parity", {})
        ok = all(par.get(k) for k in ("round", "color", "K")) if par else None
        name = NAMES[w.split("-")[0]]
        out.append(
            f"| {name} | {c['n']:,} | {c['m']:,} | {c['eps']} | {d['rounds']} | {d['jp_levels']} | "
            f"{d['colors']} | {d.get('degeneracy')} | {t:.3f} | {d['value'] / 1e9:.2f} G | "
            f"{100 * rf['path']['frac_8tbs']:.1f}% | {100 * rf['path']['frac']:.1f}% | "
            f"{100 * rf['frac']:.1f}%{'¹' if small else ''} | "
            f"{(f'{dram:.0f}' + ('¹' if small else '')) if dram is not None else '—'} | ")
        out[-1] += (f"{osec:.2f} | {cb.get('value', 0) / 1e6:.1f} M | "
                    f"{'bit-exact' if ok else ('MISMATCH' if ok is False else '—')} |") if osec else "— | — | — |"
    out.append("")
    out.append("¹ one-kernel path (csrc/small.cu): the column is that kernel (the whole path), "
               "not UPDATE.")
    print("\n".join(out))


if __name__ == "__main__":
    main()
