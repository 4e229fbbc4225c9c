"""Setup cost of the c3 1-Hash / KMV TC layouts (rank rows, orientation,
row sorting / partition), piece by piece, and the first tc_estimate call."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402

g = pg.generate_kronecker(22, 16, 2)
dev = g.device()
torch.cuda.synchronize()


def wall(label, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
    return r


for kind in ("onehash", "kmv"):
    for rep in range(2):
        sk = pg.build_sketched_graph(g, kind, s=1.0, k_override=64)
        p = pg.make_provider(kind, sketched=sk)
        dev._layouts.clear()
        dev._upper = None
        wall(f"[{kind} {rep}] degree_rank", dev.degree_rank)
        if kind == "onehash":
            wall(f"[{kind} {rep}] rank rows", p._rank_rows)
        wall(f"[{kind} {rep}] provider._tc_layout (rest)", lambda: p._tc_layout(dev))
        sk2 = pg.build_sketched_graph(g, kind, s=1.0, k_override=64)
        dev._layouts.clear()
        dev._upper = None
        wall(f"[{kind} {rep}] tc_estimate, first call (layout + pass)", lambda: pg.tc_estimate(g, sk2, kind))
        wall(f"[{kind} {rep}] tc_estimate, cached layout", lambda: pg.tc_estimate(g, sk2, kind))
        del sk, sk2, p
