"""Device time of the Bloom 1024/2 build per upload chunk vs one whole build
on a resident CSR (dev tool).   python scripts/time_chunk_builds.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200 import sketches as S  # noqa: E402
from paper_2208_11469_b200.sketches import SketchKind, BudgetPlan  # noqa: E402
from paper_2208_11469_b200 import _native as N  # noqa: E402

g = pg.generate_kronecker(20, 16, 1)
dev = g.device()
plan = BudgetPlan.explicit(SketchKind.BLOOM, g.n, bits=1024, b=2)
fam = pg.HashFamily(base_seed=0x9E3779B97F4A7C15, count=2)
seeds = torch.from_numpy(fam.seeds_array().view(np.int64)).cuda()
out = S._alloc_outputs(SketchKind.BLOOM, plan, g.n)
chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 8
targets = (np.arange(chunks + 1, dtype=np.int64) * int(g.offsets[-1])) // chunks
cuts = np.searchsorted(g.offsets, targets, side="left")
cuts[0], cuts[-1] = 0, g.n


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3


st = N.stream_handle()
print("whole", round(timed(lambda: S._launch_builders(dev, SketchKind.BLOOM, plan, seeds, out, 0, g.n, st)), 1), "us")
for c in range(chunks):
    v0, v1 = int(cuts[c]), int(cuts[c + 1])
    us = timed(lambda: S._launch_builders(dev, SketchKind.BLOOM, plan, seeds, out, v0, v1, st))
    print(f"chunk {c}: vertices {v1 - v0} entries {int(g.offsets[v1] - g.offsets[v0])} {us:.1f} us")
