"""ncu driver: one sketch build of the given kind(s) on R-MAT s20 (dev tool).
    python scripts/prof_build_once.py khash [onehash kmv bloom]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402

g = pg.generate_kronecker(20, 16, 1)
kw = {"khash": {"k_override": 32}, "onehash": {"k_override": 64}, "kmv": {"k_override": 64},
      "bloom": {"bits_override": 1024, "b": 2}}
for kind in sys.argv[1:]:
    for _ in range(2):
        sk = pg.build_sketched_graph(g, kind, s=1.0, **kw[kind])
    torch.cuda.synchronize()
    print(kind, "built")
