"""Phase breakdown of the core engine's critical path on a config graph
(PGC_PROBE build, tools/micro/build_probe.sh; stamps are %globaltimer ns).
  python tools/micro/core_probe.py [config] [key=value ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("PGC_LIB", os.path.join(ROOT, "tools", "micro", "libpgc_probe.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_2008_11321_b200 as pgc  # noqa: E402
from _refcheck import _hash_np  # noqa: E402
from bench import load_graph  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    pgc.set_tuning(k, int(v))
g = load_graph(cfg)
num, den = gg.CONFIGS[cfg][1][0]
n = g.n
off = torch.from_numpy(g.off).cuda()
col = torch.from_numpy(g.col).cuda()
a = torch.zeros(8 * n, dtype=torch.int64, device="cuda")
b = torch.zeros(n, dtype=torch.int64, device="cuda")
pgc.color_jp_adg(off, col, num, den, 1)
pgc._check(pgc._lib.pgc_debug_set_trace(a.data_ptr(), b.data_ptr(), n))
rnd, _, _, _ = pgc.color_jp_adg(off, col, num, den, 1)
st = pgc.last_stats()
pgc._check(pgc._lib.pgc_debug_set_trace(None, None, 0))
A = a.cpu().numpy().reshape(n, 8).astype(np.int64)
r = rnd.cpu().numpy().astype(np.int64)
h = _hash_np(n, 1)
NC = st["core_vertices"]
deg = np.diff(g.off)
key = np.lexsort((h, r))[::-1]
key = key[deg[key] > 0]
core = key[:NC]
incore = np.zeros(n, bool)
incore[core] = True
pub = A[:, 7]
t0 = A[core, 0].min()
# preds of core vertices (all in the core: a priority prefix is closed under pred)
cdeg = deg[core]
src = np.repeat(core, cdeg)
dst = np.concatenate([g.col[g.off[v]:g.off[v + 1]] for v in core]).astype(np.int64)
isp = (r[dst] > r[src]) | ((r[dst] == r[src]) & (h[dst] > h[src]))
src, dst = src[isp], dst[isp]
ready = np.zeros(n, np.int64)
np.maximum.at(ready, src, pub[dst])
last = np.full(n, -1, np.int64)  # the pred that completed last
order = np.argsort(pub[dst], kind="stable")
last[src[order]] = dst[order]
# critical path: from the latest-published core vertex back through the last pred
v = core[np.argmax(pub[core])]
crit = []
while v >= 0:
    crit.append(v)
    v = last[v]
crit = np.array(crit[::-1][1:])  # drop the root (no pred)
names = {0: "grab", 1: "scanned", 3: "last_pass", 4: "tail_in", 5: "tail_seen", 6: "found", 7: "pub"}
out = {"config": cfg, "core_ms": st["t_core_ms"], "crit_len": int(len(crit)),
       "span_us": float((pub[crit].max() - t0) / 1e3)}
rd = ready[crit]
step = pub[crit] - np.maximum(rd, A[crit, 0])
out["step_sum_ms"] = float(step.sum() / 1e6)
tail = A[crit, 5] != 0
out["frac_tail"] = float(tail.mean())


def pct(x):
    return [float(np.percentile(x, q)) for q in (10, 50, 90, 99)] if len(x) else []


for k, nm in names.items():
    x = A[crit, k] - rd
    ok = A[crit, k] != 0
    out[f"{nm}-ready_p10_50_90_99"] = pct(x[ok])
# classify slow hops
slow = step > 1000
out["slow_hops"] = int(slow.sum())
out["slow_sum_ms"] = float(step[slow].sum() / 1e6)
out["slow_with_tail"] = int((slow & tail).sum())
out["slow_scan_after_ready"] = int((slow & (A[crit, 1] > rd)).sum())
out["slow_lastpass_after_ready"] = int((slow & (A[crit, 3] > rd)).sum())
out["fast_step_p50"] = float(np.median(step[~slow])) if (~slow).any() else 0
print(json.dumps(out, indent=1))
# slow hops in detail: when were they grabbed, how long did their first scan take
sl = crit[slow]
npred_core = np.bincount(src, minlength=n)
det = {"grab-ready_us": pct((A[sl, 0] - ready[sl]) / 1e3), "scan_us": pct((A[sl, 1] - A[sl, 0]) / 1e3),
       "np": pct(npred_core[sl]), "fast_np": pct(npred_core[crit[~slow]]),
       "fast_scan_us": pct((A[crit[~slow], 1] - A[crit[~slow], 0]) / 1e3)}
print(json.dumps(det))
# slow hops, phase by phase (ns after ready), and whether the critical pred is local
prev = np.full(n, -1, np.int64)
prev[crit] = last[crit]
cta = {}
C = st["core_ctas"]
posc = np.full(n, -1, np.int64)
posc[core] = np.arange(NC)
def owner(v):
    p = posc[v]
    return (p // 32) % C
loc = np.array([owner(v) == owner(prev[v]) if prev[v] >= 0 else True for v in crit])
ph = {}
for nm, k in (("tail_in", 4), ("tail_seen", 5), ("found", 6), ("pub", 7), ("last_pass", 3), ("scanned", 1)):
    x = A[sl, k] - ready[sl]
    ph[nm] = pct(x[A[sl, k] != 0])
ph["local_frac_slow"] = float(loc[slow].mean()) if slow.any() else 0
ph["local_frac_fast"] = float(loc[~slow].mean())
ph["fast_step_local_p50"] = float(np.median(step[~slow & loc])) if (~slow & loc).any() else 0
ph["fast_step_remote_p50"] = float(np.median(step[~slow & ~loc])) if (~slow & ~loc).any() else 0
gap = posc[crit] - posc[np.maximum(prev[crit], 0)]
ph["gap_slow"] = pct(gap[slow])
ph["gap_fast"] = pct(gap[~slow])
ph["pos_slow"] = pct(posc[crit[slow]])
ph["pos_all"] = pct(posc[crit])
print(json.dumps(ph))
