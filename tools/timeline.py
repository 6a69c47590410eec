#!/usr/bin/env python
"""Kernel timeline of one JP-ADG step (nsys is not in the image: the CUPTI
activity trace that torch.profiler records stands in for it).  Reports, for
the step's span on the GPU: the kernel launches per stream, the busy time
(union of all kernels over both streams), the idle gaps on the call's main
stream (host syncs and launch latency show up there) and the largest gaps.

  python tools/timeline.py [--config rmat24] [--eps 1/10] [--out profiles/r2_b/timeline_rmat24.json]
"""
import argparse
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import graphgen as gg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="rmat24")
    ap.add_argument("--eps", default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import paper_2008_11321_b200 as pgc
    from bench import load_graph
    g = load_graph(a.config)
    num, den = map(int, a.eps.split("/")) if a.eps else gg.CONFIGS[a.config][1][0]
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda()
    for _ in range(3):
        pgc.color_jp_adg(off, col, num, den, 1)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        pgc.color_jp_adg(off, col, num, den, 1)
        torch.cuda.synchronize()
    st = pgc.last_stats()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    ks = [e for e in ev if e.get("cat") == "kernel" and e.get("name", "").find("pgc") >= 0]
    if not ks:
        ks = [e for e in ev if e.get("cat") == "kernel"]
    ks.sort(key=lambda e: e["ts"])
    t0 = ks[0]["ts"]
    t1 = max(e["ts"] + e["dur"] for e in ks)
    # busy = union of kernel intervals over all streams
    busy, cur_s, cur_e = 0.0, None, None
    for e in ks:
        s, f = e["ts"], e["ts"] + e["dur"]
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, f
        else:
            cur_e = max(cur_e, f)
    busy += cur_e - cur_s
    streams = {}
    for e in ks:
        streams.setdefault(e["args"].get("stream", e.get("tid")), []).append(e)
    main_stream = max(streams, key=lambda k: len(streams[k]))
    ms = streams[main_stream]
    gaps = [(ms[i + 1]["ts"] - (ms[i]["ts"] + ms[i]["dur"]), ms[i]["name"], ms[i + 1]["name"])
            for i in range(len(ms) - 1)]
    gaps_pos = [gp for gp in gaps if gp[0] > 0]
    # idle = span not covered by any kernel of any stream
    out = {
        "config": a.config, "eps": f"{num}/{den}", "span_us": t1 - t0, "busy_us": busy,
        "idle_us": (t1 - t0) - busy, "launches": len(ks),
        "launches_per_stream": {str(k): len(v) for k, v in streams.items()},
        "main_stream_gap_us": sum(gp[0] for gp in gaps_pos),
        "main_stream_gaps_over_5us": sum(1 for gp in gaps_pos if gp[0] > 5),
        "largest_gaps_us": [{"gap": round(gp[0], 1), "after": gp[1][:60], "before": gp[2][:60]}
                            for gp in sorted(gaps_pos, reverse=True)[:8]],
        "host_syncs": st["host_syncs"], "kernel_launches": st["kernel_launches"],
        "small_path": st.get("small_path", 0),
        "note": "CUPTI activity trace via torch.profiler (nsys stand-in); times in microseconds",
    }
    s = json.dumps(out, indent=1)
    print(s)
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        open(a.out, "w").write(s + "\n")


if __name__ == "__main__":
    main()
