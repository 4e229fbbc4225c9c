"""ncu driver: the Bloom 4-clique pass of config 5b (R-MAT s18 ef16 seed 4,
BF 2048/2 over N+), 2 launches.

    python scripts/prof_c5b.py
"""
import os
import sys

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
    out = four_clique_counts(view, p, 0, nnz)
torch.cuda.synchronize()
print("c5b", int(out[-1]))
