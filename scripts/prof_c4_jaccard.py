"""ncu driver: config 4 (Chung-Lu 2^23, k-Hash 32) Jaccard count, 2 launches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200.mining import jaccard_counts  # noqa: E402

g = pg.generate_chung_lu(1 << 23, 32, 2.1, 3)
sk = pg.build_sketched_graph(g, "khash", s=1.0, k_override=32)
for _ in range(2):
    c = jaccard_counts(g, sk, 0.1)
torch.cuda.synchronize()
print(c[:2].tolist())
