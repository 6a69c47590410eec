"""Per-hop breakdown of the core engine on K_n (probe build of libpgc)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["PGC_LIB"] = os.path.join(ROOT, "tools", "micro", "libpgc_probe.so")
import numpy as np, torch
import graphgen as gg
import paper_2008_11321_b200 as pgc
from _refcheck import _hash_np
n = int(sys.argv[1]); ctas = int(sys.argv[2])
g = gg.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
off = torch.from_numpy(g.off).cuda(); col = torch.from_numpy(g.col).cuda()
pgc.set_tuning("core_min_avg", 0); pgc.set_tuning("core_min_n", 1); pgc.set_tuning("core_ctas", ctas)
pgc.set_tuning("core_spin_ns", int(sys.argv[3]) if len(sys.argv) > 3 else 32)
a = torch.zeros(4 * n, dtype=torch.int64, device="cuda"); b = torch.zeros(4 * n, dtype=torch.int64, device="cuda")
pgc.color_jp_adg(off, col, 1, 10, 1)
pgc._check(pgc._lib.pgc_debug_set_trace(a.data_ptr(), b.data_ptr(), n))
r, c, T, K = pgc.color_jp_adg(off, col, 1, 10, 1)
pgc._check(pgc._lib.pgc_debug_set_trace(None, None, 0))
A = a.cpu().numpy().reshape(n, 4); B = b.cpu().numpy().reshape(n, 4)
h = _hash_np(n, 1); order = np.argsort(-h.astype(np.float64))  # priority: hash desc (all round 1)
order = np.lexsort((h,))[::-1]
A = A[order]; B = B[order]
t0 = B[:, 0].min()
A = A - t0; B = B - t0
detect, passd, mex, pub = A[:, 0], A[:, 1], A[:, 2], A[:, 3]
grab, scanned = B[:, 0], B[:, 1]
prev_pub = np.r_[0, pub[:-1]]
rows = {"pub(p-1)->last pred seen(p)": detect[1:] - prev_pub[1:], "seen->cand updated": passd - detect,
        "cand->loop exit": mex - passd, "exit->publish": pub - mex, "pub->pub": np.diff(pub),
        "grab->scanned": scanned - grab, "scanned before prev pub": prev_pub - scanned}
for k, v in rows.items():
    v = v[10:-10]
    v = v[(v > -10**7) & (v < 10**7)]
    if len(v): print(f"{k:28s} p10 {np.percentile(v,10):7.0f} p50 {np.percentile(v,50):7.0f} p90 {np.percentile(v,90):7.0f} (clock64 cycles; C=1 only)")
