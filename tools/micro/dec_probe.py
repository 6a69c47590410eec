"""DEC-ADG-ITR: passes and time on a config graph.
  python tools/micro/dec_probe.py <config> [itr_blocks_per_sm ...]"""
import sys
import time

sys.path.insert(0, '/root/repo')
import torch  # noqa: E402

import paper_2008_11321_b200 as pgc  # noqa: E402
from bench import load_graph  # noqa: E402

g = load_graph(sys.argv[1])
off = torch.from_numpy(g.off).cuda()
col = torch.from_numpy(g.col).cuda()
for bps in [int(x) for x in sys.argv[2:]] or [2]:
    pgc.set_tuning("itr_blocks_per_sm", bps)
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.time()
        r, c, T, K = pgc.color_dec_adg_itr(off, col, 1, 10, 1)
        torch.cuda.synchronize()
        best = min(best, time.time() - t)
    st = pgc.last_stats()
    print(sys.argv[1], "blocks/SM", bps, "T", T, "K", K, "passes", st["sim_col_passes"], "best ms",
          round(best * 1e3, 1), flush=True)
