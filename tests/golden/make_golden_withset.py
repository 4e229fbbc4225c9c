"""Scalar with_set and pair values from the REFERENCE (build container only):

    python tests/golden/make_golden_withset.py

For two small graphs, every sketch kind and several sizes: with_set(w, M)
(reference providers.py:164-175, 234-241, 303-307) for seeded vertices w and
member sets M of several shapes (empty, one member, a vertex's neighbourhood,
random sets beyond k, sets with repeats, members outside the graph), plus
pair(u, v) for seeded edges.  Writes withset.json.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import R, gnp  # noqa: E402

out = {}
for name, n, p, seed in (("g200", 200, 0.08, 42), ("dense120", 120, 0.6, 7)):
    g = R.CsrGraph.from_edges(gnp(n, p, seed), n=n)
    rng = np.random.default_rng(seed)
    ws = rng.integers(0, n, 12).tolist()
    sets = [[], [int(rng.integers(0, n))],
            g.adjacency[g.offsets[ws[0]]:g.offsets[ws[0] + 1]].tolist(),
            sorted(rng.choice(n, 70, replace=False).tolist()),
            sorted(rng.choice(n, 300 if n > 300 else n, replace=False).tolist()),
            [3, 3, 5, 5, 5, 9],
            [n + 5, n + 1000, 7]]
    e = g.edges()
    pairs = e[rng.choice(len(e), 20, replace=False)].tolist()
    rec = out[name] = {"n": n, "p": p, "seed": seed, "ws": ws, "sets": sets, "pairs": pairs}
    configs = [("bloom", "bf_and", {"b": 2, "bits_override": 1024}),
               ("bloom", "bf_or", {"b": 2, "bits_override": 1024}),
               ("bloom", "bf_l", {"b": 3, "bits_override": 576}),
               ("khash", "khash", {"k_override": 32}), ("khash", "khash", {"k_override": 5}),
               ("onehash", "onehash", {"k_override": 32}), ("onehash", "onehash", {"k_override": 4}),
               ("kmv", "kmv", {"k_override": 32}), ("kmv", "kmv", {"k_override": 3})]
    for skind, ekind, kw in configs:
        sk = R.build_sketched_graph(g, skind, s=1.0, seed=seed + 7, **kw)
        pv = R.make_provider(ekind, sketched=sk)
        key = f"{ekind}_{kw.get('bits_override', kw.get('k_override'))}"
        rec[key] = {"with_set": [[float(pv.with_set(w, np.asarray(m, dtype=np.int64)))
                                  for m in sets] for w in ws],
                    "pair": [float(pv.pair(u, v)) for u, v in pairs], "kw": kw, "skind": skind}
        # the scalar estimators on sketch objects (reference estimators.py)
        est = []
        for u, v in pairs[:8]:
            a, b = sk.sketch(u), sk.sketch(v)
            su, sv = int(sk.sizes[u]), int(sk.sizes[v])
            if skind == "bloom":
                est.append([R.est_intersection_bf_and(a, b), R.est_intersection_bf_limit(a, b),
                            R.est_intersection_bf_or(a, b, su, sv),
                            R.est_intersection_bf_or(a, b, su, sv, clamp=False)])
            elif skind in ("khash", "onehash"):
                est.append([R.est_jaccard_minhash(a, b), R.est_intersection_minhash(a, b, su, sv)])
            else:
                est.append([R.est_intersection_kmv(a, b, su, sv),
                            R.est_intersection_kmv(a, b, su, sv, clamp=False)])
        rec[key]["est"] = [[float(x) for x in r] for r in est]
    print(name, flush=True)
json.dump(out, open(os.path.join(HERE, "withset.json"), "w"), indent=1)
