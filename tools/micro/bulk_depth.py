import sys, numpy as np, time
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import graphgen as gg, oracle as O
from _refcheck import _hash_np
g=gg.config_graph('rmat24')
r,st=O.adg(g,1,10)
n=g.n
h=_hash_np(n,1)
deg=np.diff(g.off)
key=np.lexsort((h, r))[::-1]   # priority order: round desc, hash desc
key=key[deg[key]>0]
pos=np.full(n, -1, np.int64); pos[key]=np.arange(len(key))
c_all, K, lvl, J = O.jp(g, r, 1, levels=True)
print('J', J, 'ordered', len(key))
for P in (65535, 131072, 262144, 524288):
    core = key[:P]
    print(P, 'max level in core', int(lvl[core].max()))
    # bulk-only depth: induced subgraph on vertices with pos >= P (isolated removed anyway)
    keep = (pos >= P)
    src = np.repeat(np.arange(n), deg)
    m = keep[src] & keep[g.col]
    s2 = src[m]; d2 = g.col[m]
    cnt = np.bincount(s2, minlength=n)
    off2 = np.zeros(n+1, np.int64); np.cumsum(cnt, out=off2[1:])
    sub = gg.Graph(n, off2, d2.astype(np.int32), 'sub')
    _, _, lv2, J2 = O.jp(sub, r, 1, levels=True)
    print(P, 'bulk-only depth', J2)
