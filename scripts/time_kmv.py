import os, sys, torch
sys.path.insert(0, ".")
import paper_2208_11469_b200 as pg
from paper_2208_11469_b200.mining import tc_counts
g = pg.generate_kronecker(20, 16, 1)
for k in (32, 64):
    sk = pg.build_sketched_graph(g, "kmv", s=1.0, k_override=k)
    p = pg.make_provider("kmv", sketched=sk)
    for _ in range(2): tc_counts(p, g.device())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): c = tc_counts(p, g.device())
    b.record(); torch.cuda.synchronize()
    print(os.environ.get("PG_KMV_LANES", "default"), k, a.elapsed_time(b) / 5, p._tc_combine(c.cpu().numpy()))
