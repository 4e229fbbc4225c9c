"""Link-prediction golden values from the REFERENCE (build container only).

    python tests/golden/make_golden_linkpred.py     # ~1-2 min

For a few seeded graphs: the reference's split (make_link_prediction_split),
its two-hop candidates (checksum + count), the per-candidate
vertex_similarity scores of every (provider, measure) combination the
reference supports (checksum of the float64 bytes; the error name where it
raises) and link_prediction_eval hit counts at several top_count values.
Writes linkpred.json.  Nothing at test time reads /root/reference.
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import probgraph as R  # noqa: E402
from probgraph import mining as RM  # noqa: E402
from paper_2208_11469_b200 import graphs as G  # noqa: E402

MEASURES = ["jaccard", "overlap", "common_neighbors", "total_neighbors",
            "adamic_adar", "resource_allocation"]
PROVIDERS = {  # name -> (sketch kind or None, kwargs, estimator kind)
    "exact": (None, {}, "exact_merge"),
    "bf_and": ("bloom", {"b": 2, "bits_override": 256}, "bf_and"),
    "bf_or": ("bloom", {"b": 2, "bits_override": 256}, "bf_or"),
    "khash": ("khash", {"k_override": 16}, "khash"),
    "onehash": ("onehash", {"k_override": 16}, "onehash"),
    "kmv": ("kmv", {"k_override": 16}, "kmv"),
}
CASES = {
    "rmat8": (lambda: G.generate_kronecker(8, 8, 21, device=False), 0.2, 5),
    "er300": (lambda: G.generate_erdos_renyi_gnm(300, 1500, 6), 0.1, 7),
}
TOPS = [1, 10, 100, 1000, 10 ** 9]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


out = {}
for name, (make, frac, seed) in CASES.items():
    mine = make()
    g = R.CsrGraph(mine.offsets, mine.adjacency.astype(np.int64))
    split = R.make_link_prediction_split(g, frac, seed)
    sp = split.sparse_graph
    cands = RM._two_hop_candidates(sp)
    rec = {"n": g.n, "m": g.m, "fraction": frac, "seed": seed,
           "edges_removed": sha(split.edges_removed.astype("<i8")),
           "sparse_adjacency": sha(sp.adjacency.astype("<i8")),
           "candidates": sha(cands.astype("<i8")), "candidate_count": int(len(cands)),
           "results": {}}
    for pname, (skind, kw, ekind) in PROVIDERS.items():
        if skind is None:
            prov = R.make_provider(ekind, graph=sp)
        else:
            sk = R.build_sketched_graph(sp, skind, s=1.0, seed=seed + 1000, **kw)
            prov = R.make_provider(ekind, sketched=sk)
        for meas in MEASURES:
            key = f"{pname}/{meas}"
            try:
                sc = np.array([R.vertex_similarity(int(u), int(v), meas, prov, sp)
                               for u, v in cands.tolist()], dtype=np.float64)
                hits = [RM.link_prediction_eval(g, split, meas, prov, t) for t in TOPS]
                rec["results"][key] = {"scores": sha(sc.astype("<f8")), "hits": hits,
                                       "score_sum": float(sc.sum())}
            except Exception as ex:  # noqa: BLE001 - the reference's error is the golden
                rec["results"][key] = {"error": type(ex).__name__}
        print(name, pname, flush=True)
    out[name] = rec
json.dump(out, open(os.path.join(HERE, "linkpred.json"), "w"), indent=1)
print("wrote linkpred.json")
