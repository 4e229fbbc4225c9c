import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg
z = np.load("tests/golden/small_cases.npz")
name, k, step = sys.argv[1], int(sys.argv[2]), sys.argv[3]
g = pg.CsrGraph(z[f"{name}/offsets"], z[f"{name}/adjacency"])
sk = pg.build_sketched_graph(g, "kmv", s=1.0, seed=311, k_override=k)
p = pg.make_provider("kmv", sketched=sk)
e = g.edges()
if step == "upper":
    us, vs = g.device().upper_edges()
    torch.cuda.synchronize()
    print("upper ok", us.numel(), len(e), flush=True)
else:
    us = torch.from_numpy(e[:, 0].astype(np.int32)).cuda()
    vs = torch.from_numpy(e[:, 1].astype(np.int32)).cuda()
    out = p._tc_counts(us, vs, 0, us.numel())
    torch.cuda.synchronize()
    print("tc ok", out.item() / 3, flush=True)
