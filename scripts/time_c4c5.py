"""CUDA-event timing of the c4 Jaccard count and the c5 Bloom TC, L2 flushed
between reps (dev tool).   python scripts/time_c4c5.py [c4] [c5]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg
from paper_2208_11469_b200.mining import jaccard_counts, tc_counts

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5):
    for _ in range(2):
        out = fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); out = fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), out


tag = os.environ.get("PG_L2_WINDOW_MB", "0")
if "c4" in sys.argv:
    g = pg.generate_chung_lu(1 << 23, 32, 2.1, 3)
    sk = pg.build_sketched_graph(g, "khash", s=1.0, k_override=32)
    t, c = timed(lambda: jaccard_counts(g, sk, 0.1))
    print(f"window={tag} c4: {t:.3f} ms  {c[:2].tolist()}", flush=True)
    del g, sk
if "c5" in sys.argv:
    g = pg.generate_kronecker(24, 16, 4)
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048)
    p = pg.make_provider("bf_and", sketched=sk)
    t, c = timed(lambda: tc_counts(p, g.device()))
    print(f"window={tag} c5: {t:.3f} ms  {p._tc_combine(c.cpu().numpy()) / 3.0!r}", flush=True)
