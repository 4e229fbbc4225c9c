"""Time the fused Bloom TC kernel under the current PG_TC_* env settings.

Usage: PG_TC_ENGINE=staged PG_TC_NS=3 python scripts/sweep_tc.py --scale 20 --bits 1024
Caches the generated graph under /tmp so repeated runs in one gpurun call
skip generation.  Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--bits", type=int, default=1024)
ap.add_argument("--b", type=int, default=2)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--kind", default="bf_and")
args = ap.parse_args()

cache = f"/tmp/pg_rmat_{args.scale}_{args.ef}_{args.seed}.npz"
if os.path.exists(cache):
    z = np.load(cache)
    g = pg.CsrGraph(z["o"], z["a"])
else:
    g = pg.generate_kronecker(args.scale, args.ef, args.seed)
    np.savez(cache, o=g.offsets, a=g.adjacency)
sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=args.b, bits_override=args.bits)
p = pg.make_provider(args.kind, sketched=sk)
us, vs = g.device().upper_edges()
lus, lvs, slots, padded = p._tc_layout(g.device())
m = us.numel()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = p._tc_counts(lus, lvs, 0, slots, padded).cpu().numpy()
times = []
st = torch.cuda.current_stream()
for i in range(args.reps + 3):
    N.call("pg_l2_flush", N.ptr(flush), flush.numel(), N.stream_handle())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    out = p._tc_counts(lus, lvs, 0, slots, padded)
    b.record(st)
    torch.cuda.synchronize()
    if i >= 3:
        times.append(a.elapsed_time(b))
    assert np.array_equal(out.cpu().numpy(), ref)
ms = float(np.median(times))
print(json.dumps({"engine": os.environ.get("PG_TC_ENGINE", "staged"),
                  "ns": os.environ.get("PG_TC_NS", "3"), "minb": os.environ.get("PG_TC_MINB", ""),
                  "scale": args.scale, "bits": args.bits, "m": m, "ms": ms,
                  "gedges_s": m / ms / 1e6, "alg_gbs": m * (args.bits / 4 + 8) / ms / 1e6,
                  "estimate": p._tc_combine(ref) / 3.0}), flush=True)
