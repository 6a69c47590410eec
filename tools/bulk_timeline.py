import sys, os, json
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np, torch
import graphgen as gg, oracle as O
import paper_2008_11321_b200 as pgc
from _refcheck import _hash_np
g = gg.config_graph('rmat24'); num, den = 1, 10
off = torch.from_numpy(g.off).cuda(); col = torch.from_numpy(g.col).cuda()
tg = torch.zeros(g.n, dtype=torch.int64, device='cuda'); td = torch.zeros(g.n, dtype=torch.int64, device='cuda')
pgc.color_jp_adg(off, col, num, den, 1)
pgc.set_tuning('timing', 1)
pgc.debug_set_trace(tg, td)
r, c, T, K = pgc.color_jp_adg(off, col, num, den, 1)
st = pgc.last_stats(); pgc.debug_set_trace(None, None)
tg = tg.cpu().numpy(); td = td.cpu().numpy(); r = r.cpu().numpy()
# npred per vertex
deg = np.diff(g.off); n = g.n; h = _hash_np(n, 1)
src = np.repeat(np.arange(n, dtype=np.int64), deg); dst = g.col.astype(np.int64)
isp = (r[dst] > r[src]) | ((r[dst] == r[src]) & (h[dst] > h[src]))
npred = np.bincount(src[isp], minlength=n); del src, dst, isp
key = np.lexsort((h, r))[::-1]; core = np.zeros(n, bool); core[key[:st['core_vertices']]] = True
traced = td > 0
t0 = tg[traced].min()
out = {'core_ms': st['t_core_ms'], 'jp_ms': st['t_jp_ms']}
for name, m in [('core', core & traced), ('heavy', (~core) & (npred > 62) & traced), ('light', (~core) & (npred >= 1) & (npred <= 62) & traced)]:
    if m.sum() == 0: continue
    d = (td[m] - t0) / 1e3; gr = (tg[m] - t0) / 1e3
    out[name] = {'n': int(m.sum()), 'grab_us_p0_50_100': [float(np.percentile(gr, q)) for q in (0, 50, 100)],
                 'done_us_p0_10_50_90_100': [float(np.percentile(d, q)) for q in (0, 10, 50, 90, 100)],
                 'done_minus_grab_p50_us': float(np.percentile(d - gr, 50))}
    for R in range(1, T + 1):
        mr = m & (r == R)
        if mr.sum(): out[name][f'round{R}_done_us_p50_100'] = [float(np.percentile((td[mr]-t0)/1e3, q)) for q in (50, 100)] + [int(mr.sum())]
print(json.dumps(out, indent=1))
