#!/usr/bin/env python
"""bench.py -- JP-ADG (ADG ordering + Jones-Plassmann coloring) on B200.

Metric (BASELINE.json): JP-ADG edges/sec (ADG+JP, 1 B200) and % HBM roofline;
#colors.  One "step" = one full pgc_color_jp_adg call (every SURVEY.md §8(a)
row: init, ADG rounds with fused JP Part 1, priority order, JP coloring) on a
device-resident synthetic graph.  Default workload: R-MAT scale 24, edge
factor 16, eps = 1/10 (BASELINE.json configs[3], the headline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config rmat24] [--impl pgc|reference]

N > 1 runs one independent replica per GPU (the path does not shard, DESIGN.md
"Multi-GPU"): value = total edges colored by all ranks / max-over-ranks time.
The reference arm (--impl reference) times the CPU oracle (oracle/), as it
stands, on a bounded sample of the workload (see REF_SAMPLE).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import graphgen as gg  # noqa: E402  (input harness: no method arithmetic)

METRIC = "JP-ADG edges/sec (ADG+JP, 1 B200) and % HBM roofline; #colors"
REF_SAMPLE = {"rmat24": ("rmat22", lambda: gg.rmat(22, 16, seed=1))}
PROFILES = os.path.join(ROOT, "profiles")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["pgc", "reference"], default="pgc")
    ap.add_argument("--config", default="rmat24", choices=sorted(gg.CONFIGS))
    ap.add_argument("--eps", default=None, help="num/den (default: the config's first eps)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip e2e, cpu baseline (for ncu runs)")
    ap.add_argument("--serial-schedule", action="store_true",
                    help="one stream (tuning jp_split_overlap=0): for ncu launch lists, which "
                         "serialise kernels anyway (the overlapped schedule would make the core "
                         "rewrite its lists itself there)")
    ap.add_argument("--method", choices=["jp-adg", "jp-adg-m", "jp-adg-o", "jp-r", "jp-ff", "jp-lf",
                                         "jp-llf", "dec-adg-itr", "adg-push", "adg-pull"],
                    default="jp-adg",
                    help="jp-adg-m: the median variant (SURVEY.md §8(f) NEXT-3, PAPER.md:2273-2303); "
                         "jp-adg-o: ADG-O's total order (NEXT-1, PAPER.md:2397-2453); "
                         "jp-r/ff/lf/llf: the JP baselines (NEXT-4, PAPER.md:1093-1103); "
                         "dec-adg-itr: DEC-ADG-ITR (NEXT-2, PAPER.md:1957-1972); "
                         "adg-push/adg-pull: the ADG ordering alone with the push or pull "
                         "(CREW) UPDATE (NEXT-4, PAPER.md:2331-2342)")
    return ap.parse_args()


def eps_of(args):
    if args.eps:
        a, b = args.eps.split("/")
        return int(a), int(b)
    return gg.CONFIGS[args.config][1][0]


# ------------------------------------------------------------------ graph ---
def _gen_hash():
    h = hashlib.sha1(open(os.path.join(ROOT, "graphgen", "graphgen.c"), "rb").read())
    h.update(open(os.path.join(ROOT, "graphgen", "__init__.py"), "rb").read())
    return h.hexdigest()[:12]


def load_graph(name, local_rank=0, barrier=None):
    """Generate the config graph; ranks of one node share it via a /tmp cache
    (setup only -- no timing or result depends on the cache)."""
    path = f"/tmp/pgc_graph_{name}_{_gen_hash()}.npz"
    if local_rank == 0 and not os.path.exists(path):
        g = gg.config_graph(name)
        tmp = path + f".{os.getpid()}.tmp.npz"
        np.savez(tmp, off=g.off, col=g.col)
        os.replace(tmp, path)
    if barrier:
        barrier()
    if local_rank == 0 and name in gg._cache:
        return gg._cache[name]
    z = np.load(path)
    return gg.Graph(int(len(z["off"]) - 1), z["off"], z["col"], name)


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            # warm NVML up first (its first calls can take tens of ms), so the
            # samples cover the timed region that follows
            try:
                self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 1.0:
                time.sleep(0.001)
            self.samples.clear()   # keep only samples taken inside the region
            self.reasons.clear()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": [],
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ model ---
def survey_bytes(n, nnz, m, X, sum_active):
    """Algorithmic bytes of SURVEY.md §8(d) (per-touch model: each logical
    access once at its size, no sector inflation, no cache credit), with JP
    Part 1 fused into UPDATE at zero extra bytes:
      init 20n | ADG scans 12 sum_l n_l | per removed vertex 16n |
      ADG arcs 8 nnz + 8X | JP per vertex 20n | JP arcs 8 nnz + 12m
    B_alg = 44m + 8X + 12 sum_l n_l + 56n (nnz = 2m)."""
    t = {"init": 20 * n, "adg_scans": 12 * sum_active, "adg_vertex": 16 * n,
         "adg_arcs": 8 * nnz + 8 * X, "jp_vertex": 20 * n, "jp_arcs": 8 * nnz + 12 * m}
    t["update"] = t["adg_arcs"] + t["adg_vertex"]       # row a4 (+ its per-vertex term)
    t["path"] = 44 * m + 8 * X + 12 * sum_active + 56 * n
    assert t["path"] == sum(t[k] for k in ("init", "adg_scans", "adg_vertex", "adg_arcs",
                                           "jp_vertex", "jp_arcs"))
    return t


def builder_bytes(n, nnz, m, X, sum_active):
    """The builder's own per-group model (round 1), kept for context only: it
    also charges this design's pred-list stores (4m) and record traffic."""
    return {
        "init": 8 * n + 12 * n,
        "select": 12 * sum_active + 20 * n,
        "update": 24 * n + 8 * nnz + 8 * X + 4 * m,
        "order": 56 * n,
        "jp": 20 * n + 8 * m,
    }


def peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_traffic(workload):
    """DRAM bytes (ncu dram__bytes_read.sum + dram__bytes_write.sum) of one
    step's UPDATE launches on THIS workload, from profiles/traffic.json
    (written by tools/traffic.py from an ncu pass over the same path and
    workload); None when that workload was never captured."""
    try:
        d = json.load(open(os.path.join(PROFILES, "traffic.json")))
        e = d.get(workload)
        return (e["update_dram_bytes_per_step"], e["source"]) if e else (None, None)
    except Exception:
        return None, None


def host_info():
    model, mhz = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name") and model is None:
                model = line.split(":", 1)[1].strip()
            if line.startswith("cpu MHz") and mhz is None:
                mhz = float(line.split(":", 1)[1])
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "cpu_mhz": mhz}


def step_stats(times_ms):
    """median, min, mean and the 95% CI of the mean (t quantile; the paper's
    reporting)."""
    k = len(times_ms)
    mean = statistics.mean(times_ms)
    sd = statistics.stdev(times_ms) if k > 1 else 0.0
    tq = {1: 12.71, 2: 4.30, 3: 3.18, 4: 2.78, 5: 2.57, 6: 2.45, 7: 2.36, 8: 2.31, 9: 2.26,
          10: 2.23, 15: 2.13, 20: 2.09, 30: 2.04}
    df = max(1, k - 1)
    q = tq.get(df) or tq[min(tq, key=lambda d: abs(d - df))]
    half = q * sd / (k ** 0.5) if k > 1 else 0.0
    return {"median_ms": statistics.median(times_ms), "min_ms": min(times_ms), "mean_ms": mean,
            "ci95_ms": [mean - half, mean + half], "steps": k}


# ------------------------------------------------------------- multi-GPU ----
def reduce_max_ms(ms, dist, device):
    """Step time of the whole job = the slowest rank (N independent replicas,
    DESIGN.md "Multi-GPU"); identity without torch.distributed."""
    if dist is None:
        return ms
    import torch
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_value(world, m, ms):
    """Whole-job throughput: every rank colors its own copy of the graph."""
    return world * m / (ms * 1e-3)


# ------------------------------------------------------------------ arms ----
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    num, den = eps_of(args)
    sample_name, make = REF_SAMPLE.get(args.config, (args.config, lambda: gg.config_graph(args.config)))
    g = make()
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r, _ = O.adg(g, num, den)
        O.jp(g, r, args.seed)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = statistics.mean(times)
    v = g.m / t
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "edges/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
           "data": "synthetic",
           "config": {"workload": f"{args.config}-eps{num}/{den}", "sample": sample_name,
                      "eps": f"{num}/{den}", "seed": args.seed},
           "cpu_baseline": {"value": v, "unit": "edges/s", "cores": 1, "kind": "oracle",
                            "sample": f"sequential C oracle (oracle/oracle.c), full JP-ADG on the "
                                      f"{sample_name} graph (same recipe, eps, seed) per step"},
           "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def run_pgc(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    barrier = (lambda: dist.barrier()) if dist else None

    import paper_2008_11321_b200 as pgc

    num, den = eps_of(args)
    g = load_graph(args.config, local_rank, barrier)
    n, nnz, m = g.n, g.nnz, g.m
    dev = torch.device("cuda", local_rank)
    off = torch.from_numpy(g.off).to(dev)
    col = torch.from_numpy(g.col).to(dev)
    rnd = torch.empty(n, dtype=torch.int32, device=dev)
    color = torch.empty(n, dtype=torch.int32, device=dev)

    median = args.method == "jp-adg-m"
    sortedR = args.method == "jp-adg-o"
    baseline = args.method in ("jp-r", "jp-ff", "jp-lf", "jp-llf")
    decitr = args.method == "dec-adg-itr"
    adgonly = args.method in ("adg-push", "adg-pull")

    def step():
        if adgonly:
            r_, T_ = pgc.adg_order(off, col, num, den, update=args.method[4:], round_out=rnd)
            return r_, color, T_, 0
        if decitr:
            return pgc.color_dec_adg_itr(off, col, num, den, args.seed, round_out=rnd, color_out=color)
        if baseline:
            c_, K_ = pgc.jp_baseline(off, col, args.method, args.seed, color_out=color)
            return rnd, c_, 0, K_
        if median:
            return pgc.color_jp_adg_m(off, col, args.seed, round_out=rnd, color_out=color)
        if sortedR:
            return pgc.color_jp_adg_o(off, col, num, den, round_out=rnd, color_out=color)
        return pgc.color_jp_adg(off, col, num, den, args.seed, round_out=rnd, color_out=color)

    pgc.set_tuning("timing", 0)
    # ablation hook: PGC_TUNE="key=value,key=value" (library tuning knobs)
    for kv in filter(None, os.environ.get("PGC_TUNE", "").split(",")):
        k, v = kv.split("=")
        pgc.set_tuning(k.strip(), int(v))
    if args.serial_schedule:
        pgc.set_tuning("jp_split_overlap", 0)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)

    # ---- timed region A: the headline (no per-launch events) ----
    # an event between consecutive steps gives per-step times (each call blocks
    # until its stream is idle, so the events add nothing to a step)
    launches = 0
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local_rank) as clk:
        if barrier:
            barrier()
        torch.cuda.synchronize()
        evs[0].record(stream)
        for i in range(args.steps):
            _, _, T, K = step()
            launches += pgc.last_stats()["kernel_launches"]
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        if barrier:
            barrier()
    ms = reduce_max_ms(evs[0].elapsed_time(evs[-1]) / args.steps, dist, dev)
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    st = pgc.last_stats()

    # ---- timed region B: same steps with per-launch CUDA events (attribution) ----
    pgc.set_tuning("timing", 1)
    groups = {"t_select_ms": [], "t_update_ms": [], "t_adg_other_ms": [], "t_order_ms": [],
              "t_core_ms": [], "t_jp_ms": [], "t_total_ms": []}
    for _ in range(args.steps):
        step()
        s = pgc.last_stats()
        for k in groups:
            groups[k].append(s[k])
    pgc.set_tuning("timing", 0)
    gmean = {k: statistics.mean(v) for k, v in groups.items()}

    # ---- J (JP levels): one more, untimed call with the levels pass on ----
    J = None
    if not (adgonly or decitr):
        pgc.set_tuning("levels", 1)
        step()
        J = pgc.last_stats()["jp_levels"]
        pgc.set_tuning("levels", 0)

    X, sum_active = st["cross_edges"], st["sum_active"]
    sv = survey_bytes(n, nnz, m, X, sum_active)
    model = builder_bytes(n, nnz, m, X, sum_active)
    upd_arcs = nnz   # arcs UPDATE classifies per step
    upd_bytes = sv["update"]
    path_bytes = sv["path"]
    path_model = "SURVEY 8(d): B_alg = 44m + 8X + 12 sum_l n_l + 56n"
    if adgonly:
        # ADG alone: init, scans, per-vertex and arcs terms of 8(d) (no JP rows)
        path_bytes = sv["init"] + sv["adg_scans"] + sv["adg_vertex"] + sv["adg_arcs"]
        path_model = "SURVEY 8(d) ADG rows: 20n + 12 sum_l n_l + 16n + 8 nnz + 8X"
        if args.method == "adg-pull":
            # pull: every survivor rescans its adjacency: sum_v (round[v]-1) * deg(v) arcs,
            # a col read + a state gather each, one D update per survivor per round
            r_h = rnd.cpu().numpy().astype(np.int64)
            pull_arcs = int(((r_h - 1) * g.degrees().astype(np.int64)).sum())
            upd_bytes = 8 * pull_arcs + 8 * sum_active
            path_bytes = sv["init"] + sv["adg_scans"] + sv["adg_vertex"] + upd_bytes
            upd_arcs = pull_arcs
    peak, peak_kind = peak_gbs()
    t_upd = gmean["t_update_ms"]
    small = bool(st.get("small_path", 0))
    if small:
        # one persistent kernel runs the whole path (csrc/small.cu): its dominant
        # (only) kernel is charged the whole path's 8(d) bytes
        t_upd = gmean["t_select_ms"]
        upd_bytes = path_bytes
    achieved = upd_bytes / (t_upd * 1e-3) / 1e9
    workload = (f"{args.config}-{args.method}" if (baseline or decitr or adgonly) else
                f"{args.config}-adgm" if median else
                f"{args.config}-adgo-eps{num}/{den}" if sortedR else f"{args.config}-eps{num}/{den}")
    traffic, traffic_src = measured_traffic(workload)
    if small:   # the profiles' UPDATE traffic does not apply: the step is one other kernel
        traffic, traffic_src = measured_traffic(workload + "-small")
    # the builder's uniform-target probe of the gather+RED mix (context, not a ceiling:
    # UPDATE beats it because hub targets hit in L2)
    ra = None
    try:
        pr = json.load(open(os.path.join(PROFILES, "random_access_probe.json")))
        arcs_per_s = upd_arcs / (t_upd * 1e-3)
        key = "gather_u8_per_s" if args.method == "adg-pull" else "gather_plus_red_42pct_arcs_per_s"
        ra = {"arcs_per_s": arcs_per_s, "red_fraction": 0.0 if args.method == "adg-pull" else
              (X / upd_arcs if upd_arcs else 0.0),
              "uniform_probe_arcs_per_s": pr[key], "ratio_to_uniform_probe": arcs_per_s / pr[key],
              "note": "tools/micro/atom_probe.cu: uniformly random targets on a 16.7 M-vertex "
                      "state; NOT a ceiling for skewed (R-MAT) targets"}
    except Exception:
        pass

    out = {
        "metric": (METRIC.replace("JP-ADG", "JP-ADG-M").replace("ADG+JP", "ADG-M+JP") if median else
                   METRIC.replace("JP-ADG", "JP-ADG-O").replace("ADG+JP", "ADG-O+JP") if sortedR else
                   METRIC.replace("JP-ADG", args.method.upper()).replace("ADG+JP", "JP only")
                   if baseline else
                   METRIC.replace("JP-ADG", "DEC-ADG-ITR").replace("ADG+JP", "ADG+SIM-COL-ITR")
                   if decitr else
                   METRIC.replace("JP-ADG", args.method.upper()).replace("ADG+JP", "ordering only")
                   .replace("; #colors", "") if adgonly else METRIC),
        "value": job_value(world, m, ms), "unit": "edges/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": workload,
                   "method": args.method, "n": n, "m": m, "nnz": nnz,
                   "eps": f"{num}/{den}", "seed": args.seed, "graph_seed": 1,
                   "parallelism": f"replicas{world}" if world > 1 else "single-gpu",
                   "l2": ("inputs larger than L2 (CSR %.2f GB vs 126 MB L2); no flush" %
                          ((8 * (n + 1) + 4 * nnz) / 1e9)) if 8 * (n + 1) + 4 * nnz > 126e6 else
                         ("CSR %.1f MB fits the 126 MB L2: steps run back to back with a warm L2 "
                          "(this small config is latency-bound, not bandwidth-bound)" %
                          ((8 * (n + 1) + 4 * nnz) / 1e6))},
        "timing": step_stats(per_step),
        "colors": K, "rounds": T, "jp_levels": J, "cross_edges": X, "sum_active": sum_active,
        "core_vertices": st["core_vertices"], "core_ctas": st["core_ctas"],
        "small_path": int(st.get("small_path", 0)),
        "roofline": {"bound": "hbm",
                     "kernel": ("k_small_jp_adg: the whole JP-ADG in ONE persistent cooperative "
                                "kernel (%d grid barriers: 1 + 2T + J)" % (1 + 2 * T + (J or 0))
                                if small else
                                "ADG UPDATE with fused JP Part 1 (k_update_light + k_update_heavy + "
                                "k_update_heavy_f, every round of one step)"),
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes": upd_bytes, "ms_per_launch": t_upd,
                     "bytes_model": (path_model if small else
                                     "SURVEY 8(d) rows a4: 8 nnz + 8X, plus the 16n per-removed-"
                                     "vertex term" if args.method != "adg-pull" else
                                     "pull: 8 bytes per rescanned arc + 8 per survivor-round"),
                     "path": {"bytes": path_bytes, "model": path_model,
                              "achieved_gbs": path_bytes / (ms * 1e-3) / 1e9,
                              "frac": path_bytes / (ms * 1e-3) / 1e9 / peak,
                              "frac_8tbs": path_bytes / (ms * 1e-3) / 8e12},
                     "builder_model": {"update_bytes": model["update"],
                                       "path_bytes": sum(model.values()),
                                       "note": "round-1 builder model incl. pred-list stores (4m); "
                                               "context only"},
                     "random_access": ra},
        "breakdown_ms": {k[2:-3]: v for k, v in gmean.items()},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }

    # ---- end to end through the host-buffer C-ABI call ----
    if not (args.no_e2e or args.quick or median or sortedR or baseline or decitr or adgonly):
        h_off = torch.from_numpy(g.off).pin_memory()
        h_col = torch.from_numpy(g.col).pin_memory()
        h_r = torch.empty(n, dtype=torch.int32).pin_memory()
        h_c = torch.empty(n, dtype=torch.int32).pin_memory()
        pgc.color_jp_adg_host(h_off, h_col, num, den, args.seed, h_r, h_c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if barrier:
            barrier()
        e0.record(stream)
        for _ in range(args.steps):
            pgc.color_jp_adg_host(h_off, h_col, num, den, args.seed, h_r, h_c)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = reduce_max_ms(e0.elapsed_time(e1) / args.steps, dist, dev)
        out["e2e"] = {"value": job_value(world, m, ems), "unit": "edges/s",
                      "h2d_bytes_per_step": 8 * (n + 1) + 4 * nnz, "d2h_bytes_per_step": 8 * n,
                      "ms_per_step": ems}
        parity_ok = bool(torch.equal(h_r, rnd.cpu()) and torch.equal(h_c, color.cpu()))
        out["e2e"]["matches_device_api"] = parity_ok

    # ---- CPU oracle baseline (rank 0, N=1) + parity of this run ----
    if rank == 0 and world == 1 and not (args.no_cpu_baseline or args.quick):
        import oracle as O
        t0 = time.perf_counter()
        if baseline:
            import math
            deg = g.degrees()
            r_or = {"jp-r": np.zeros(n), "jp-ff": -np.arange(n), "jp-lf": deg,
                    "jp-llf": np.array([math.ceil(math.log2(d)) if d > 1 else 0 for d in deg])
                    }[args.method].astype(np.int32)
        elif sortedR:
            r_or, rho, _, _, _ = O.adg_o(g, num, den)
        else:
            r_or, _ = O.adg_m(g) if median else O.adg(g, num, den)
        t1 = time.perf_counter()
        if adgonly:
            c_or, K_or = color.cpu().numpy(), K   # no coloring: only round[] is checked
        elif decitr:
            c_or, K_or, _ = O.dec_adg_itr(g, r_or, args.seed)
        else:
            c_or, K_or = O.jp_rho(g, rho) if sortedR else O.jp(g, r_or, args.seed)
        t2 = time.perf_counter()
        t3 = time.perf_counter()
        out["degeneracy"] = O.degeneracy(g)     # d (exact, Matula-Beck peel)
        t_d = time.perf_counter() - t3
        out["cpu_baseline"] = {"value": m / (t2 - t0), "unit": "edges/s", "cores": 1,
                               "kind": "oracle", "host": host_info(),
                               "oracle_ms": {"adg": (t1 - t0) * 1e3, "jp": (t2 - t1) * 1e3,
                                             "degeneracy": t_d * 1e3},
                               "sample": f"full {args.config} workload, one "
                                         f"{'ADG' if adgonly else 'JP-ADG'} run of the "
                                         f"sequential C oracle (ADG {t1 - t0:.1f}s + greedy JP "
                                         f"{t2 - t1:.1f}s)"}
        out["parity"] = {"round": True if baseline else bool(np.array_equal(rnd.cpu().numpy(), r_or)),
                         "color": bool(np.array_equal(color.cpu().numpy(), c_or)),
                         "K": K == K_or}
        if J is not None and not sortedR:   # J of the oracle's greedy (untimed, after the baseline)
            _, _, _, J_or = O.jp(g, r_or, args.seed, levels=True)
            out["parity"]["J"] = J == J_or

    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_pgc(args)


if __name__ == "__main__":
    sys.exit(main())
