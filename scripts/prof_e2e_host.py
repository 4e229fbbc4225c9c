"""cProfile of the public-API e2e path (host CSR -> estimate) at c2: where
the host time goes around the pipelined upload."""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("PG_REPO", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2208_11469_b200 as pg  # noqa: E402

g = pg.generate_kronecker(20, 16, 1)


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t


off_h, adj_h = pinned(g.offsets).numpy(), pinned(g.adjacency.astype(np.int32)).numpy()


def e2e():
    gr = pg.CsrGraph(off_h, adj_h)
    sk = pg.build_sketched_graph(gr, "bloom", s=1.0, b=2, bits_override=1024)
    return pg.tc_estimate(gr, sk, "bf_and")


for _ in range(3):
    e2e()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    e2e()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
