"""Setup cost of the degree-oriented c5 TC layout, piece by piece."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402

g = pg.generate_kronecker(24, 16, 4)
dev = g.device()
torch.cuda.synchronize()


def wall(label, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
    return r


for rep in range(2):
    dev._layouts.clear()
    wall(f"[{rep}] degree_rank", dev.degree_rank)
    wall(f"[{rep}] hub_slots(8, 0)", lambda: dev.hub_slots(8, 0))
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048)
    p = pg.make_provider("bf_and", sketched=sk)
    dev._layouts.clear()
    wall(f"[{rep}] provider._tc_layout", lambda: p._tc_layout(dev))
    dev._layouts.clear()
    wall(f"[{rep}] tc_estimate (layout + pass)", lambda: pg.tc_estimate(g, sk, "bf_and"))
    wall(f"[{rep}] tc_estimate (cached layout)", lambda: pg.tc_estimate(g, sk, "bf_and"))
