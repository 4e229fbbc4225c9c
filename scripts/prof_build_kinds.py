"""Per-kernel device times of one sketch build per kind at c3 scale (dev tool)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg
from torch.profiler import ProfilerActivity, profile

g = pg.generate_kronecker(22, 16, 2)
g.device()
for kind in sys.argv[1:] or ["onehash", "kmv"]:
    pg.build_sketched_graph(g, kind, s=1.0, k_override=64)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        pg.build_sketched_graph(g, kind, s=1.0, k_override=64)
        torch.cuda.synchronize()
    print(kind)
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=8, max_name_column_width=60))
