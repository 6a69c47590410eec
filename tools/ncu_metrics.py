#!/usr/bin/env python
"""Selected raw metrics of every launch in an ncu report: ncu_metrics.py rep [substr ...]"""
import csv
import subprocess
import sys

DEFAULT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_sector_hit_rate.pct", "lts__t_requests.sum",
           "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed",
           "lts__t_tag_requests.max.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum",
           "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
           "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "l1tex__throughput.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_lg_throttle",
           "smsp__pcsamp_warps_issue_stalled_membar", "smsp__pcsamp_warps_issue_stalled_drain",
           "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_wait",
           "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
           "smsp__pcsamp_warps_issue_stalled_branch_resolving", "smsp__pcsamp_warps_issue_stalled_no_instruction",
           "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_warps_issue_stalled_selected",
           "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_sample_count"]


def main():
    rep = sys.argv[1]
    want = sys.argv[2:] or DEFAULT
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for v in rows[2:]:
        print("==", v[h.index("Kernel Name")][:60] if "Kernel Name" in h else "")
        for i, k in enumerate(h):
            if any(k == w or (w.endswith("*") and k.startswith(w[:-1])) for w in want):
                print(f"  {k:70s} {v[i]}")


if __name__ == "__main__":
    main()
