"""ncu driver: config 5 (R-MAT s24, Bloom 2048/2) fused TC, 2 launches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200.mining import tc_counts  # noqa: E402

g = pg.generate_kronecker(24, 16, 4)
sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048)
p = pg.make_provider("bf_and", sketched=sk)
for _ in range(2):
    c = tc_counts(p, g.device())
torch.cuda.synchronize()
print(p._tc_combine(c.cpu().numpy()) / 3.0)
