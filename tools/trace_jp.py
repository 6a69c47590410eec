#!/usr/bin/env python
"""JP dataflow diagnostics from per-vertex %globaltimer stamps (pgc_debug.h).

For every vertex: grab time, done time, and `ready` = the done time of its
last predecessor.  Reports the chain pace (done time per JP level, levels from
the oracle), and the step latency t_done - ready for heavy / light vertices.
  python tools/trace_jp.py --config rmat20
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle as O  # noqa: E402
from _refcheck import _hash_np  # noqa: E402


def pct(a, qs=(50, 90, 99, 100)):
    if len(a) == 0:
        return {}
    return {f"p{q}": float(np.percentile(a, q)) for q in qs}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="rmat20")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--tune", nargs="*", default=[], help="key=value tuning knobs")
    a = ap.parse_args()
    import paper_2008_11321_b200 as pgc
    for kv in a.tune:
        k, val = kv.split("=")
        pgc.set_tuning(k, int(val))
    from bench import load_graph  # /tmp-cached generator output
    g = load_graph(a.config)
    num, den = gg.CONFIGS[a.config][1][0] if a.config != "rmat20" else (1, 10)
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda()
    tg = torch.zeros(g.n, dtype=torch.int64, device="cuda")
    td = torch.zeros(g.n, dtype=torch.int64, device="cuda")
    pgc.color_jp_adg(off, col, num, den, a.seed)   # warm
    pgc.set_tuning("timing", 1)
    pgc.debug_set_trace(tg, td)
    rnd, color, T, K = pgc.color_jp_adg(off, col, num, den, a.seed)
    st = pgc.last_stats()
    pgc.debug_set_trace(None, None)
    tg = tg.cpu().numpy().astype(np.int64)
    td = td.cpu().numpy().astype(np.int64)
    r = rnd.cpu().numpy().astype(np.int64)
    traced = td > 0              # isolated vertices are settled before JP (no stamps)
    t0 = tg[traced].min()
    tg = np.where(traced, tg - t0, 0)
    td = np.where(traced, td - t0, 0)
    # oracle levels (JP DAG depth)
    _, _, lvl, J = O.jp(g, rnd.cpu().numpy(), a.seed, levels=True)
    # pred relation and ready time = max done over preds
    n = g.n
    deg = np.diff(g.off)
    h = _hash_np(n, a.seed)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    dst = g.col.astype(np.int64)
    is_pred = (r[dst] > r[src]) | ((r[dst] == r[src]) & (h[dst] > h[src]))
    npred = np.bincount(src[is_pred], minlength=n)
    val = np.where(is_pred, td[dst], -1)
    ready = np.full(n, -1, dtype=np.int64)
    nz = deg > 0
    ready[nz] = np.maximum.reduceat(val, g.off[:-1][nz])
    del src, dst, is_pred, val
    heavy = npred > 62
    has_pred = npred > 0
    # core = the first core_vertices positions of the priority order
    key = np.lexsort((h, r))[::-1]          # round desc, then hash desc
    core = np.zeros(n, dtype=bool)
    core[key[:st["core_vertices"]]] = True
    step = td - np.maximum(ready, tg)
    wait_grab = tg - ready  # >0: the vertex was grabbed after it became ready
    out = {"config": a.config, "tune": a.tune, "n": n, "J": J, "T": T, "K": K,
           "jp_ms": st["t_jp_ms"], "span_ms": float(td.max() / 1e6),
           "heavy": int(heavy.sum()), "core_vertices": int(core.sum()),
           "core_ms": st["t_core_ms"]}
    # chain pace: time when each level finished (max done over the level)
    lv_done = np.zeros(J + 1, dtype=np.int64)
    np.maximum.at(lv_done, lvl, td)
    lv_done = np.maximum.accumulate(lv_done)
    marks = sorted(set([1, 10, 100, J // 4, J // 2, 3 * J // 4, J - 50, J - 10, J]))
    out["level_done_us"] = {int(L): float(lv_done[L] / 1e3) for L in marks if 0 < L <= J}
    out["ns_per_level"] = float(lv_done[J] / max(J, 1))
    for name, m in (("core", core & has_pred), ("heavy", heavy & has_pred & ~core),
                    ("light", ~heavy & has_pred & ~core)):
        out[f"step_ns_{name}"] = pct(step[m])
        out[f"grab_after_ready_ns_{name}"] = pct(wait_grab[m])
        out[f"done_minus_grab_ns_{name}"] = pct((td - tg)[m])
    # critical path: walk back from a vertex of level J through the latest pred
    crit = []
    v = int(np.argmax(lvl))
    off_np = g.off
    for _ in range(J):
        crit.append(v)
        nb = g.col[off_np[v]:off_np[v + 1]].astype(np.int64)
        pm = (r[nb] > r[v]) | ((r[nb] == r[v]) & (h[nb] > h[v]))
        if not pm.any():
            break
        preds = nb[pm]
        v = int(preds[np.argmax(td[preds])])
    crit = np.array(crit[::-1])
    cs = step[crit]
    cc = core[crit]
    late = wait_grab[crit] > 0   # grabbed after it was ready: its whole scan is on the path
    out["critical_core_late_grab"] = {"n": int((cc & late).sum()),
                                      "sum_grab_after_ready_ms": float(wait_grab[crit][cc & late].sum() / 1e6),
                                      "sum_step_ms": float(cs[cc & late].sum() / 1e6),
                                      "step_ns": pct(cs[cc & late])}
    out["critical_core_early_grab"] = {"n": int((cc & ~late).sum()),
                                       "sum_step_ms": float(cs[cc & ~late].sum() / 1e6),
                                       "step_ns": pct(cs[cc & ~late], (10, 50, 90, 99, 100))}
    out["critical_core"] = {"len": int(cc.sum()), "step_ns": pct(cs[cc]), "sum_step_ms": float(cs[cc].sum() / 1e6),
                            "grab_after_ready_sum_ms": float(np.maximum(wait_grab[crit][cc], 0).sum() / 1e6),
                            "span_ms": float((td[crit][cc].max() - tg[crit][cc].min()) / 1e6) if cc.any() else 0}
    nb = ~cc
    out["critical_bulk"] = {"len": int(nb.sum()), "step_ns": pct(cs[nb]), "sum_step_ms": float(cs[nb].sum() / 1e6),
                            "grab_after_ready_sum_ms": float(np.maximum(wait_grab[crit][nb], 0).sum() / 1e6)}
    out["critical"] = {"len": len(crit), "step_ns": pct(cs), "heavy_frac": float(heavy[crit].mean()),
                       "rounds": np.bincount(r[crit]).tolist(),
                       "sum_step_ms": float(cs.sum() / 1e6),
                       "grab_after_ready_sum_ms": float(np.maximum(wait_grab[crit], 0).sum() / 1e6)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
