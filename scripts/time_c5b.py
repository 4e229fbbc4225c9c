"""CUDA-event timing of the 4-clique Bloom 2048/2 pass on R-MAT s18 seed 4 (c5b; dev tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200.mining import four_clique_counts  # noqa: E402

g = pg.generate_kronecker(18, 16, 4)
view = pg.degree_order(g)
dsk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048, source="directed", view=view)
p = pg.make_provider("bf_and", sketched=dsk)
nnz = view.device().nnz
for _ in range(2):
    c = four_clique_counts(view, p, 0, nnz)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    c = four_clique_counts(view, p, 0, nnz)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
c = c.cpu().numpy()
print(f"c5b: {np.median(ts):.3f} ms  triples {int(c[-1])}  estimate {p._tc_combine(c[:-1])!r}")
