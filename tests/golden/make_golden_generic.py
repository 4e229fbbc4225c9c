"""Golden values for sketch sizes beyond the tuned kernels (Bloom rows over
32,768 / 65,536 bits, k > 256), from the REFERENCE (build container only):

    python tests/golden/make_golden_generic.py

plan_budget (reference sketches.py:115-138) gives such sizes on dense
graphs (B = s*(n+2m)/n*64, k = s*2m/n); the explicit overrides here pin them
on small G(n, p) graphs.  Arrays are recorded as sha256 of their canonical
little-endian bytes (the full matrices are megabytes), scalars as values.
Writes generic.json.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import R, canon, gnp  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


out = {}
# dense graph: avg degree ~150; plan_budget(s=1) would give k ~ 150, B ~ 9.7k
name, n, p, seed = "dense300", 300, 0.5, 21
g = R.CsrGraph.from_edges(gnp(n, p, seed), n=n)
e = g.edges()
us, vs = e[:, 0], e[:, 1]
rec = out[name] = {"n": n, "p": p, "seed": seed, "m": int(g.m)}
for bits, b in ((40000, 2), (70016, 2), (65600, 1)):
    sk = R.build_sketched_graph(g, "bloom", s=1.0, b=b, bits_override=bits)
    key = f"bloom{bits}_{b}"
    rec[key] = {k2: sha(v2) for k2, v2 in canon(sk).items()}
    for kind in ("bf_and", "bf_l", "bf_or"):
        pv = R.make_provider(kind, sketched=sk)
        rec[key][f"pairs_{kind}"] = sha(pv.pair_many(us, vs).astype("<f8"))
        rec[key][f"tc_{kind}"] = R.tc_estimate(g, sk, kind)
    print(key, flush=True)
for k in (300, 513):
    for kind in ("khash", "onehash", "kmv"):
        sk = R.build_sketched_graph(g, kind, s=1.0, k_override=k)
        key = f"{kind}{k}"
        rec[key] = {k2: sha(v2) for k2, v2 in canon(sk).items()}
        pv = R.make_provider(kind, sketched=sk)
        rec[key]["pairs"] = sha(pv.pair_many(us, vs).astype("<f8"))
        rec[key]["tc"] = R.tc_estimate(g, sk, kind)
        jp = R.jarvis_patrick_cluster(g, pv, 50.0)
        rec[key]["jp50"] = [len(jp.kept_edges), jp.cluster_count, jp.singleton_count]
        if kind == "khash":
            jh = np.array([R.est_jaccard_minhash(sk.sketch(int(a)), sk.sketch(int(c)))
                           for a, c in zip(us, vs)])
            js = np.array([R.vertex_similarity(int(a), int(c), "jaccard", pv, g)
                           for a, c in zip(us, vs)])
            rec[key]["kept_jhat_ge_0.1"] = int(np.count_nonzero(jh >= 0.1))
            rec[key]["kept_sim_ge_0.1"] = int(np.count_nonzero(js >= 0.1))
        print(key, flush=True)

# 4-clique on a sparser graph with the same wide sketches over N+
name, n, p, seed = "c4g120", 120, 0.35, 5
g = R.CsrGraph.from_edges(gnp(n, p, seed), n=n)
view = R.degree_order(g)
rec = out[name] = {"n": n, "p": p, "seed": seed}
for kind, k in (("khash", 300), ("onehash", 300), ("kmv", 300), ("onehash", 40), ("kmv", 40)):
    dsk = R.build_sketched_graph(g, kind, s=1.0, k_override=k, source="directed", view=view)
    rec[f"{kind}{k}_dir"] = float(R.four_clique_count(view, R.make_provider(kind, sketched=dsk)))
    print(name, kind, k, flush=True)
for bits in (70016, 20032):
    dsk = R.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=bits, source="directed",
                                 view=view)
    for kind in ("bf_and", "bf_or"):
        rec[f"bloom{bits}_{kind}_dir"] = float(
            R.four_clique_count(view, R.make_provider(kind, sketched=dsk)))
    print(name, bits, flush=True)

json.dump(out, open(os.path.join(HERE, "generic.json"), "w"), indent=1)
