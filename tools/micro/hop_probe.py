"""Per-hop phase breakdown of the core engine on K_n (PGC_PROBE build of libpgc,
tools/micro/build_probe.sh).  Stamps are SM clock64 cycles, so use ctas=1.
  python tools/micro/hop_probe.py <n> <ctas> [core_spin_ns]"""
import os, sys
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
pgc.set_tuning("core_spin_ns", int(sys.argv[3]) if len(sys.argv) > 3 else 1024)
a = torch.zeros(8 * n, dtype=torch.int64, device="cuda"); b = torch.zeros(8 * n, dtype=torch.int64, device="cuda")
pgc.color_jp_adg(off, col, 1, 10, 1)
pgc._check(pgc._lib.pgc_debug_set_trace(a.data_ptr(), b.data_ptr(), n))
pgc.color_jp_adg(off, col, 1, 10, 1)
pgc._check(pgc._lib.pgc_debug_set_trace(None, None, 0))
A = a.cpu().numpy().reshape(n, 8).astype(np.int64)
h = _hash_np(n, 1)
A = A[np.lexsort((h,))[::-1]]          # priority order (all in one round): hash desc
names = ["grab", "scanned", "-", "last pass", "tail in", "tail seen", "found", "published"]
pub = A[:, 7]
def pr(label, v):
    v = v[20:-20]
    v = v[(v > -10**8) & (v < 10**8)]
    if len(v): print(f"{label:34s} p10 {np.percentile(v,10):7.0f} p50 {np.percentile(v,50):7.0f} p90 {np.percentile(v,90):7.0f}  (n={len(v)})")
pr("pub(p-1) -> pub(p)", np.diff(pub))
for k in (1, 3, 4, 5, 6):
    has = A[1:, k] != 0
    pr(f"pub(p-1) -> {names[k]}(p)", np.where(has, A[1:, k] - pub[:-1], -10**9))
pr("tail in -> tail seen", np.where(A[:, 4] != 0, A[:, 5] - A[:, 4], -10**9))
pr("tail seen -> published", np.where(A[:, 5] != 0, A[:, 7] - A[:, 5], -10**9))
print("vertices with tail:", int((A[:, 5] != 0).sum()), "of", n)
