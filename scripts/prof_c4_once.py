"""ncu driver: 4-clique Bloom 2048/2 on R-MAT s18 seed 4 (c5b), 2 launches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402

g = pg.generate_kronecker(18, 16, 4)
view = pg.degree_order(g)
dsk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048, source="directed", view=view)
p = pg.make_provider("bf_and", sketched=dsk)
for _ in range(2):
    est = pg.four_clique_count(view, p)
torch.cuda.synchronize()
print("4-clique bf_and", est)
