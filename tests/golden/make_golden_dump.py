"""PGSKETCH v1 files written by the REFERENCE (build container only).

    python tests/golden/make_golden_dump.py

Sketches of a small seeded R-MAT graph for every kind (undirected, and one
directed Bloom set), dumped with the reference's dump_sketches into
tests/golden/pgsketch/*.bin (a few KB each).  Tests check that this package
writes byte-identical files and reads these back exactly.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import probgraph as R  # noqa: E402
from paper_2208_11469_b200 import graphs as G  # noqa: E402

mine = G.generate_kronecker(7, 8, 3, device=False)
g = R.CsrGraph(mine.offsets, mine.adjacency.astype(np.int64))
out = os.path.join(HERE, "pgsketch")
os.makedirs(out, exist_ok=True)
cases = {
    "bloom_576_3": dict(kind="bloom", s=1.0, b=3, bits_override=576, seed=11),
    "bloom_budget": dict(kind="bloom", s=0.5, b=2, seed=12),
    "khash_16": dict(kind="khash", s=1.0, k_override=16, seed=13),
    "onehash_8": dict(kind="onehash", s=1.0, k_override=8, seed=14),
    "kmv_8": dict(kind="kmv", s=1.0, k_override=8, seed=15),
}
for name, kw in cases.items():
    kind = kw.pop("kind")
    sk = R.build_sketched_graph(g, kind, **kw)
    R.dump_sketches(sk, os.path.join(out, name + ".bin"))
view = R.degree_order(g)
sk = R.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=256, seed=16, source="directed", view=view)
R.dump_sketches(sk, os.path.join(out, "bloom_directed.bin"))
print(sorted(os.listdir(out)))

# reference results on the same sketches, for the plugin-boundary tests
# (tests/test_gpu_plugin_boundary.py): tc_estimate per estimator, per-edge
# pair_many doubles, the 4-clique count over the directed Bloom sketches
import hashlib  # noqa: E402
import json  # noqa: E402

est_kinds = {"bloom": ["bf_and", "bf_l", "bf_or"], "khash": ["khash"], "onehash": ["onehash"],
             "kmv": ["kmv"]}
e = g.edges()
expected = {"graph": "generate_kronecker(7, 8, 3)", "m": int(g.m)}
for name in cases:
    ld = R.load_sketches(os.path.join(out, name + ".bin"))
    for kind in est_kinds[ld.kind.value]:
        p = R.make_provider(kind, sketched=ld)
        pm = p.pair_many(e[:, 0], e[:, 1])
        expected[f"{name}/{kind}"] = {
            "tc_estimate": R.tc_estimate(g, ld, kind),
            "pair_many_sha": hashlib.sha256(np.ascontiguousarray(pm, "<f8").tobytes()).hexdigest()}
ld = R.load_sketches(os.path.join(out, "bloom_directed.bin"))
expected["bloom_directed/four_clique_count"] = R.four_clique_count(
    view, R.make_provider("bf_and", sketched=ld))
with open(os.path.join(out, "expected.json"), "w") as fh:
    json.dump(expected, fh, indent=1)
print(expected)
