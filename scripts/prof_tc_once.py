"""Minimal driver for ncu: c2 graph + Bloom sketches, a few TC launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402

bits = int(os.environ.get("BITS", "1024"))
scale = int(os.environ.get("SCALE", "20"))
cache = f"/tmp/pg_rmat_{scale}_16_1.npz"
if os.path.exists(cache):
    z = np.load(cache)
    g = pg.CsrGraph(z["o"], z["a"])
else:
    g = pg.generate_kronecker(scale, 16, 1)
    np.savez(cache, o=g.offsets, a=g.adjacency)
sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=bits)
p = pg.make_provider("bf_and", sketched=sk)
us, vs = g.device().upper_edges()
lus, lvs, slots, padded = p._tc_layout(g.device())
for _ in range(4):
    out = p._tc_counts(lus, lvs, 0, slots, padded)
torch.cuda.synchronize()
print("tc", p._tc_combine(out.cpu().numpy()) / 3.0)
