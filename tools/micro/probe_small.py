import sys, torch
sys.path.insert(0, '.')
import graphgen as gg, paper_2008_11321_b200 as pgc
pgc.set_tuning('small_max_arcs', 1 << 40); pgc.set_tuning('small_max_avg', 1 << 30)
for name in sys.argv[1:]:
    g = gg.config_graph(name); num, den = gg.CONFIGS[name][1][0]
    off = torch.from_numpy(g.off).cuda(); col = torch.from_numpy(g.col).cuda()
    for _ in range(3): pgc.color_jp_adg(off, col, num, den, 1)
    torch.cuda.synchronize(); print(name, pgc.last_stats()['rounds'], flush=True)
