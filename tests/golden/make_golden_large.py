"""Large-config golden values from the REFERENCE (build container only).

    python tests/golden/make_golden_large.py   # ~20-40 min, ~40 GB RAM

Graphs come from this repo's host generators (bit-identical to the
reference's generate_kronecker, checked in make_golden.py); sketches and
estimates from the unmodified reference package.  Writes large.json.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import probgraph as R  # noqa: E402
from paper_2208_11469_b200 import graphs as G  # noqa: E402

out_path = os.path.join(HERE, "large.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}


def save():
    json.dump(res, open(out_path, "w"), indent=1)


def ref_graph(g):
    return R.CsrGraph(g.offsets, g.adjacency.astype(np.int64))


which = sys.argv[1:] or ["c3", "c4", "c5b", "c5"]
if "c3" in which:
    g = ref_graph(G.generate_kronecker(22, 16, 2, device=False))
    for kind in ("onehash", "kmv"):
        t = time.time()
        sk = R.build_sketched_graph(g, kind, s=1.0, k_override=64)
        v = R.tc_estimate(g, sk, kind, threads=8)
        res[f"c3_{kind}64_tc"] = {"graph": "rmat s22 ef16 seed2", "m": g.m, "value": v,
                                  "seconds": time.time() - t}
        save()
        print(kind, v, flush=True)
        del sk
    del g
if "c4" in which:
    g = ref_graph(G.generate_chung_lu(1 << 23, 32, 2.1, 3, device=False))
    t = time.time()
    sk = R.build_sketched_graph(g, "khash", s=1.0, k_override=32)
    e = g.edges()
    m = np.empty(len(e), dtype=np.int64)
    for lo in range(0, len(e), 1 << 21):
        hi = min(lo + (1 << 21), len(e))
        a, c = sk.entries[e[lo:hi, 0]], sk.entries[e[lo:hi, 1]]
        m[lo:hi] = np.count_nonzero((a == c) & (a >= 0), axis=1)
    res["c4_khash32"] = {"graph": "chung-lu 2^23 avg32 g2.1 seed3", "m": g.m,
                         "match_hist": np.bincount(m, minlength=33).tolist(),
                         "kept_jhat_ge_0.1": int(np.count_nonzero(m / 32 >= 0.1)),
                         "tc_khash": R.tc_estimate(g, sk, "khash", threads=8),
                         "seconds": time.time() - t}
    save()
    print("c4", res["c4_khash32"]["kept_jhat_ge_0.1"], flush=True)
    del sk, g, e, m
if "c5b" in which:
    g = ref_graph(G.generate_kronecker(18, 16, 4, device=False))
    view = R.degree_order(g)
    sk = R.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048, source="directed",
                                view=view)
    # full with_set over a fixed 1% sample of directed edges (seed 0): the
    # reference's own functions, histogram of popcounts
    p = R.make_provider("bf_and", sketched=sk)
    src = np.repeat(np.arange(view.n), view.out_degrees())
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(len(src), size=len(src) // 100, replace=False))
    t = time.time()
    total = 0.0
    trip = 0
    for j in sample.tolist():
        u, v = int(src[j]), int(view.adjacency[j])
        c3 = R.setops.intersect_members(view.out_neighbors(u), view.out_neighbors(v))
        for w in c3.tolist():
            total += p.with_set(w, c3)
            trip += 1
    ex = R.make_provider("exact_merge", view=view)
    np.savez_compressed(os.path.join(HERE, "c5b_sample.npz"), edge_ids=sample.astype(np.int64))
    res["c5b_4clique_sample"] = {"graph": "rmat s18 ef16 seed4 directed", "sample_seed": 0,
                                 "sample_file": "c5b_sample.npz", "triples": trip,
                                 "bf_and_sum": total, "seconds": time.time() - t,
                                 "exact_tc": R.triangle_count(view, ex, threads=8)}
    save()
    print("c5b", trip, total, flush=True)
if "c5" in which:
    g = ref_graph(G.generate_kronecker(24, 16, 4, device=False))
    t = time.time()
    sk = R.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048)
    v = R.tc_estimate(g, sk, "bf_and", threads=8)
    res["c5_bloom2048_tc"] = {"graph": "rmat s24 ef16 seed4", "m": g.m, "bf_and": v,
                              "seconds": time.time() - t}
    save()
    print("c5", v, flush=True)
