"""ncu driver: s20 graph, 1-Hash k=64 and KMV k=64 fused TC, 2 launches each."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg
from paper_2208_11469_b200.mining import tc_counts
cache = "/tmp/pg_rmat_20_16_1.npz"
if os.path.exists(cache):
    z = np.load(cache); g = pg.CsrGraph(z["o"], z["a"])
else:
    g = pg.generate_kronecker(20, 16, 1); np.savez(cache, o=g.offsets, a=g.adjacency)
for kind in sys.argv[1:]:
    sk = pg.build_sketched_graph(g, kind, s=1.0, k_override=64)
    p = pg.make_provider(kind, sketched=sk)
    for _ in range(2):
        out = tc_counts(p, g.device())
    torch.cuda.synchronize()
    print(kind, p._tc_combine(out.cpu().numpy()) / 3.0)
