"""ncu driver: config 1 (ER 16384/262144, Bloom 512/1) fused TC, 3 launches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200.mining import tc_counts  # noqa: E402

g = pg.generate_erdos_renyi_gnm(16384, 262144, 0)
sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=1, bits_override=512)
p = pg.make_provider("bf_and", sketched=sk)
for _ in range(3):
    c = tc_counts(p, g.device())
torch.cuda.synchronize()
print(p._tc_combine(c.cpu().numpy()) / 3.0)
