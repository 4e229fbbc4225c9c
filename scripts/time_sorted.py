"""CUDA-event timing of the fused 1-Hash / KMV TC kernels (dev tool).

    python scripts/time_sorted.py SCALE SEED kind [kind ...]
"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg
from paper_2208_11469_b200.mining import tc_counts

scale, seed = int(sys.argv[1]), int(sys.argv[2])
g = pg.generate_kronecker(scale, 16, seed)
dev = g.device()
for kind in sys.argv[3:]:
    sk = pg.build_sketched_graph(g, kind, s=1.0, k_override=64)
    p = pg.make_provider(kind, sketched=sk)
    for _ in range(2):
        out = tc_counts(p, dev)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = tc_counts(p, dev)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = float(np.median(ts))
    print(f"{kind} s{scale}: {t:.3f} ms  {g.m / t / 1e6:.2f} G edges/s  est {p._tc_combine(out.cpu().numpy()) / 3.0!r}",
          flush=True)
