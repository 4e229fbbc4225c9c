"""CUDA-event timings of every device path on one graph (dev tool).

    python scripts/time_all.py [--scale 20] [--c4scale 18]
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
from paper_2208_11469_b200.graphs import DeviceCsr  # noqa: E402
from paper_2208_11469_b200.mining import tc_counts  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--c4scale", type=int, default=18)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()


def graph(scale, seed):
    cache = f"/tmp/pg_rmat_{scale}_16_{seed}.npz"
    if os.path.exists(cache):
        z = np.load(cache)
        return pg.CsrGraph(z["o"], z["a"])
    g = pg.generate_kronecker(scale, 16, seed)
    np.savez(cache, o=g.offsets, a=g.adjacency)
    return g


def timed(fn, reps=args.reps):
    st = torch.cuda.current_stream()
    out = fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        out = fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), out


res = {}
g = graph(args.scale, args.seed)
m = g.m
res["graph"] = {"scale": args.scale, "n": g.n, "m": m}
dev = g.device()


def fresh_upper():
    d = DeviceCsr.__new__(DeviceCsr)
    d.__dict__.update(dev.__dict__)
    d._upper, d._layouts = None, {}
    return d.upper_edges()


res["upper_edges_ms"], _ = timed(fresh_upper)
for kind, kw, est in (("bloom", dict(b=2, bits_override=1024), "bf_and"),
                      ("bloom", dict(b=2, bits_override=2048), "bf_and"),
                      ("khash", dict(k_override=32), "khash"),
                      ("onehash", dict(k_override=64), "onehash"),
                      ("kmv", dict(k_override=64), "kmv")):
    tag = f"{kind}{kw.get('bits_override', kw.get('k_override'))}"
    tb, sk = timed(lambda: pg.build_sketched_graph(g, kind, s=1.0, **kw))
    p = pg.make_provider(est, sketched=sk)
    tt, counts = timed(lambda: tc_counts(p, dev))
    r = {"build_ms": tb, "tc_ms": tt, "tc_gedges_s": m / tt / 1e6,
         "estimate": p._tc_combine(counts.cpu().numpy()) / 3.0}
    if kind == "khash":
        tj, jc = timed(lambda: pg.jaccard_cluster_count(g, sk, 0.1))
        r["jaccard_ms"] = tj
        r["jaccard_kept"] = [jc.kept_hat, jc.kept_similarity]
    res[tag] = r
    print(tag, json.dumps(r), flush=True)
    del sk, p

g4 = graph(args.c4scale, 4)
view = pg.degree_order(g4)
dsk = pg.build_sketched_graph(g4, "bloom", s=1.0, b=2, bits_override=2048, source="directed",
                              view=view)
pb = pg.make_provider("bf_and", sketched=dsk)
t4, v4 = timed(lambda: pg.four_clique_count(view, pb), reps=2)
ex = pg.make_provider("exact_merge", view=view)
t4e, v4e = timed(lambda: pg.four_clique_count(view, ex), reps=2)
ttc, tce = timed(lambda: pg.triangle_count(view, ex), reps=2)
from paper_2208_11469_b200.mining import four_clique_counts  # noqa: E402
c = four_clique_counts(view, pb, 0, view.device().nnz).cpu().numpy()
res["clique4"] = {"scale": args.c4scale, "bloom_ms": t4, "estimate": v4, "exact_ms": t4e,
                  "exact": v4e, "triples": int(c[-1]), "triples_per_s": int(c[-1]) / t4 * 1e3,
                  "exact_tc_ms": ttc, "exact_tc": tce}
print(json.dumps(res), flush=True)
