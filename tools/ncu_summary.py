#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration per launch) and an optional
`ncu --set full` report into a markdown table + JSON (profiles/<round>/).

  python tools/ncu_summary.py gpurun_out/r1b profiles/r1
"""
import collections
import csv
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_atom.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_requests.sum", "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed",
        "lts__t_tag_requests.max.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum"]


def short(name):
    return name.split("(")[0].replace("void ", "").strip()


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    steps = []
    for r in rows[hi + 1:]:
        name = short(r[ki])
        t = float(r[vi].replace(",", ""))
        if name in ("k_adg_init", "k_adg_state_init"):
            steps.append(collections.OrderedDict())
        if steps:
            steps[-1].setdefault(name, [0.0, 0])
            steps[-1][name][0] += t
            steps[-1][name][1] += 1
    return steps


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {units[h.index(k)]}".strip()
        res.append(d)
    return res


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    md = []
    summary = {}
    lp = os.path.join(src, "launches.csv")
    if os.path.exists(lp):
        steps = launches(lp)
        # the last TIMED step: bench.py's extra untimed call with the levels
        # pass (k_jp_levels, J) comes after the timed steps and is skipped
        timed = [st for st in steps if "k_jp_levels" not in st]
        last = (timed or steps)[-1]
        tot = sum(v[0] for v in last.values())
        md.append(f"## Launch list (last timed step of `{os.path.basename(src)}`; ncu "
                  f"gpu__time_duration, cold-cache, serialised; the untimed levels call "
                  f"is excluded)\n")
        md.append("| kernel | launches | ms | share |\n|---|---|---|---|")
        for k, (t, c) in sorted(last.items(), key=lambda x: -x[1][0]):
            md.append(f"| {k} | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
        md.append(f"| **total** | {sum(v[1] for v in last.values())} | {tot / 1e6:.3f} | |\n")
        summary["launch_list_last_step"] = {k: {"ns": t, "launches": c} for k, (t, c) in last.items()}
    import glob
    fl = []
    for rp in sorted(glob.glob(os.path.join(src, "*.ncu-rep"))):
        fl += full(rp)
    if fl:
        summary["full"] = fl
        md.append("## ncu --set full (selected launches)\n")
        for d in fl:
            md.append(f"### {d['kernel']}\n")
            for k in KEYS:
                if k in d:
                    md.append(f"- {k}: {d[k]}")
            md.append("")
    open(os.path.join(dst, "ncu_summary.md"), "w").write("\n".join(md) + "\n")
    json.dump(summary, open(os.path.join(dst, "ncu_summary.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
