"""1-Hash / KMV TC pass time at k = 32, 64, 128 on R-MAT s20 (engine
sanity check across the supported sizes); engines follow the PG_* knobs."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200.mining import tc_counts  # noqa: E402

g = pg.generate_kronecker(20, 16, 1)
for kind in ("onehash", "kmv"):
    for k in (32, 64, 128):
        sk = pg.build_sketched_graph(g, kind, s=1.0, k_override=k)
        p = pg.make_provider(kind, sketched=sk)
        for _ in range(2):
            out = tc_counts(p, g.device())
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = tc_counts(p, g.device())
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(kind, k, f"{statistics.median(ts):.3f} ms", p._tc_combine(out.cpu().numpy()) / 3.0, flush=True)
        del sk, p
