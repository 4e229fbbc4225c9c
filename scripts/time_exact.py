"""CUDA-event timing of the exact triangle count (directed view, exact
provider) and the exact 4-clique count (dev tool)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg


def timed(fn, reps=3):
    out = fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); out = fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), out


for scale, seed in ((20, 1), (18, 4)):
    g = pg.generate_kronecker(scale, 16, seed)
    view = pg.degree_order(g)
    ex = pg.make_provider("exact_merge", view=view)
    t, tri = timed(lambda: pg.triangle_count(view, ex))
    print(f"s{scale}: exact triangles {tri} in {t:.2f} ms", flush=True)
    if scale == 18:
        t, c4 = timed(lambda: pg.four_clique_count(view, ex))
        print(f"s{scale}: exact 4-cliques {c4} in {t:.2f} ms", flush=True)
