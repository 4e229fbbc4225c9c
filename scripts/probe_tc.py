"""Bloom TC engine variants on the device: ID- vs degree-oriented slot
schedule (PG_TC_ORIENT) under the process's PG_TC_CSA / PG_TC_VCACHE /
PG_TC_MINB knobs; CUDA-event medians with an L2 flush before every call.
    python scripts/probe_tc.py [c5|c2] [orient ...]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200 import _native as N  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
orients = sys.argv[2:] or ["id", "degree"]
scale, seed, bits = {"c5": (24, 4, 2048), "c2": (20, 1, 1024), "s22": (22, 2, 2048)}[cfg]
g = pg.generate_kronecker(scale, 16, seed)
sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=bits)
p = pg.make_provider("bf_and", sketched=sk)
dev = g.device()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def tm(fn, reps=9):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        N.call("pg_l2_flush", N.ptr(flush), flush.numel(), N.stream_handle())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out


knobs = " ".join(f"{k}={os.environ[k]}" for k in sorted(os.environ) if k.startswith("PG_"))
ref = None
for o in orients:
    os.environ["PG_TC_ORIENT"] = o
    lay = p._tc_layout(dev)
    ms, h = tm(lambda: p._tc_counts_layout(lay, 0, lay.slots))
    ref = h if ref is None else ref
    print(f"{cfg} {o:6s} {knobs}: {ms:.3f} ms  {g.m / ms / 1e6:.1f} G/s  slots={lay.slots} "
          f"same={torch.equal(h, ref)}", flush=True)
