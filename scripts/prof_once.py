"""ncu driver: one BASELINE config's estimator pass at full size, 2 launches.

    python scripts/prof_once.py c3onehash|c3kmv|c4|c5|c2
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200.mining import jaccard_counts, tc_counts  # noqa: E402

cfg = sys.argv[1]
if cfg in ("c3onehash", "c3kmv"):
    g = pg.generate_kronecker(22, 16, 2)
    kind = cfg[2:]
    sk = pg.build_sketched_graph(g, kind, s=1.0, k_override=64)
    p = pg.make_provider(kind, sketched=sk)
    run = lambda: tc_counts(p, g.device())  # noqa: E731
elif cfg == "c4":
    g = pg.generate_chung_lu(1 << 23, 32, 2.1, 3)
    sk = pg.build_sketched_graph(g, "khash", s=1.0, k_override=32)
    run = lambda: jaccard_counts(g, sk, 0.1)  # noqa: E731
elif cfg in ("c5", "c2"):
    sc, seed, bits = (24, 4, 2048) if cfg == "c5" else (20, 1, 1024)
    g = pg.generate_kronecker(sc, 16, seed)
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=bits)
    p = pg.make_provider("bf_and", sketched=sk)
    run = lambda: tc_counts(p, g.device())  # noqa: E731
else:
    sys.exit(f"unknown config {cfg}")
for _ in range(2):
    out = run()
torch.cuda.synchronize()
print(cfg, out.cpu().numpy()[:4].tolist())
