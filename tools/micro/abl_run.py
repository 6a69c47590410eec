"""Runner for ablation builds of libpgc (PGC_LIB=...): two JP-ADG calls on
R-MAT 24 under a short watchdog, errors tolerated (an ablated library computes
wrong results on purpose).  Used under ncu to time k_update_light round 1 with
its state gathers, REDs or pred stores compiled out (temporary -DPGC_ABL_*
switches in Arc::raw / Arc::classify / k_update_light, not kept in the source;
results in DESIGN.md section 4, UPDATE row)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2008_11321_b200 as pgc
from bench import load_graph
g = load_graph("rmat24")
off = torch.from_numpy(g.off).cuda(); col = torch.from_numpy(g.col).cuda()
pgc.set_tuning("jp_watchdog_ms", 500)
for _ in range(2):
    try:
        pgc.color_jp_adg(off, col, 1, 10, 1)
    except Exception as e:
        print("err", e)
    torch.cuda.synchronize()
