"""4-clique golden values with k-Hash / 1-Hash / KMV providers and the
exact provider bound to the undirected graph, from the REFERENCE
(build container only):

    python tests/golden/make_golden_c4sketch.py

For every small G(n,p) graph of make_golden.SMALL, every k in KS and every
MinHash / KMV kind: ``four_clique_count(view, make_provider(kind,
sketched=build_sketched_graph(g, kind, source="directed", view=view)))``
(reference mining.py:133-154, providers.py:234-241, 303-307); plus the
exact count with ``ExactProvider.for_graph(g)`` (N(w) undirected,
providers.py:117-118) and with undirected sketches.  A larger R-MAT case
(s12, seed 4) pins a graph with hub out-lists, and an R-MAT s16 1%
directed-edge sample (seed 0) reproduces the reference's per-edge loop over
the sample (same with_set calls, summed in the reference's order).
Writes c4sketch.json.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import KS, R, SMALL, G, gnp  # noqa: E402

out = {"small": {}, "rmat": {}}
for name, n, p, seed in SMALL:
    g = R.CsrGraph.from_edges(gnp(n, p, seed), n=n)
    view = R.degree_order(g)
    rec = out["small"][name] = {}
    rec["exact_for_graph"] = int(R.four_clique_count(view, R.make_provider("exact_merge", graph=g)))
    for k in KS:
        for kind in ("khash", "onehash", "kmv"):
            t = time.time()
            dsk = R.build_sketched_graph(g, kind, s=1.0, seed=seed + 400, k_override=k,
                                         source="directed", view=view)
            rec[f"{kind}{k}_dir"] = float(R.four_clique_count(view, R.make_provider(kind, sketched=dsk)))
            if k == 32:
                usk = R.build_sketched_graph(g, kind, s=1.0, seed=seed + 500, k_override=k)
                rec[f"{kind}{k}_undir"] = float(
                    R.four_clique_count(view, R.make_provider(kind, sketched=usk)))
            print(name, kind, k, rec[f"{kind}{k}_dir"], f"{time.time() - t:.1f}s", flush=True)

# R-MAT s12 ef16 seed 4 (hub out-lists up to a few hundred), whole graph
h = G.generate_kronecker(12, 16, 4, device=False)
g = R.CsrGraph(h.offsets, h.adjacency.astype(np.int64))
view = R.degree_order(g)
rec = out["rmat"]["s12"] = {"graph": "rmat s12 ef16 seed 4", "max_out_degree":
                            int(np.diff(view.offsets).max())}
for kind, k in (("khash", 16), ("onehash", 16), ("kmv", 16)):
    t = time.time()
    dsk = R.build_sketched_graph(g, kind, s=1.0, k_override=k, source="directed", view=view)
    rec[f"{kind}{k}_dir"] = float(R.four_clique_count(view, R.make_provider(kind, sketched=dsk)))
    print("s12", kind, rec[f"{kind}{k}_dir"], f"{time.time() - t:.1f}s", flush=True)

# R-MAT s16 ef16 seed 4, 1% directed-edge sample (seed 0), k = 64
h = G.generate_kronecker(16, 16, 4, device=False)
g = R.CsrGraph(h.offsets, h.adjacency.astype(np.int64))
view = R.degree_order(g)
src = np.repeat(np.arange(view.n), np.diff(view.offsets))
sample = np.sort(np.random.default_rng(0).choice(len(src), size=len(src) // 100, replace=False))
rec = out["rmat"]["s16_sample"] = {"graph": "rmat s16 ef16 seed 4", "sample_seed": 0,
                                   "sample_size": int(len(sample))}
for kind in ("khash", "onehash", "kmv"):
    t = time.time()
    dsk = R.build_sketched_graph(g, kind, s=1.0, k_override=64, source="directed", view=view)
    pv = R.make_provider(kind, sketched=dsk)
    total, trip = 0.0, 0
    for j in sample.tolist():
        u, v = int(src[j]), int(view.adjacency[j])
        c3 = R.setops.intersect_members(view.out_neighbors(u), view.out_neighbors(v))
        for w in c3.tolist():
            total += pv.with_set(w, c3)
            trip += 1
    rec[f"{kind}64_sum"] = total
    rec["triples"] = trip
    print("s16 sample", kind, total, trip, f"{time.time() - t:.1f}s", flush=True)

json.dump(out, open(os.path.join(HERE, "c4sketch.json"), "w"), indent=1)
