import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg
z = np.load("tests/golden/small_cases.npz")
name, k, b, e = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
g = pg.CsrGraph(z[f"{name}/offsets"], z[f"{name}/adjacency"])
sk = pg.build_sketched_graph(g, "kmv", s=1.0, seed=311, k_override=k)
p = pg.make_provider("kmv", sketched=sk)
ed = g.edges()
us = torch.from_numpy(ed[:, 0].astype(np.int32)).cuda()
vs = torch.from_numpy(ed[:, 1].astype(np.int32)).cuda()
e = min(e, us.numel())
out = p._tc_counts(us, vs, b, e)
torch.cuda.synchronize()
pairs = p.pair_many(ed[b:e, 0], ed[b:e, 1])
print(name, k, b, e, "tc ok", out.item(), pairs.sum(), flush=True)
