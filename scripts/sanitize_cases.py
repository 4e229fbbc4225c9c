"""Small cases that launch every kernel family of the engine once, for
compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py

Builders incl. the hub passes (R-MAT s14: hubs of degree > 1024), the fused
Bloom / k-Hash / 1-Hash / KMV passes (ID- and degree-oriented layouts),
per-pair kernels, Jarvis-Patrick components, the 4-clique kernels (Bloom
staged and global paths, exact, MinHash / KMV sketch kernel incl. its
global-scratch path), exact TC, the device generators and link prediction.
Each result is checked against the host oracle where one is cheap.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from oracle import oracle as O  # noqa: E402

g = pg.generate_kronecker(14, 16, 3)
assert int(np.diff(g.offsets).max()) > 1024, "need hub vertices"
us, vs = O.upper_edges(g.offsets, g.adjacency)

# builders + fused passes + pairs
for bits, b in ((1024, 2), (2048, 2), (576, 3)):
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=b, bits_override=bits)
    rows, ones = O.C.build_bloom(g.offsets, g.adjacency, bits, b)
    assert np.array_equal(sk.bit_matrix, rows)
    for kind in ("bf_and", "bf_or"):
        p = pg.make_provider(kind, sketched=sk)
        pg.tc_estimate(g, sk, kind)
        p.pair_many(us[:5000], vs[:5000])
for orient in ("degree", "id"):
    os.environ["PG_TC_ORIENT"] = orient
    sk = pg.build_sketched_graph(g, "khash", s=1.0, k_override=32)
    assert np.array_equal(sk.entries, O.C.build_khash(g.offsets, g.adjacency, 32))
    pg.tc_estimate(g, sk, "khash")
    pg.jaccard_cluster_count(g, sk, 0.1)
os.environ.pop("PG_TC_ORIENT")
for kind in ("onehash", "kmv"):
    for k in (16, 64):
        sk = pg.build_sketched_graph(g, kind, s=1.0, k_override=k)
        p = pg.make_provider(kind, sketched=sk)
        pg.tc_estimate(g, sk, kind)
        p.pair_many(us[:5000], vs[:5000])
        pg.jarvis_patrick_cluster(g, p, 1.0)

# 4-clique: Bloom (staged + global), exact (view and graph rows), sketches
view = pg.degree_order(g)
for bits in (2048, 576):
    dsk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=bits, source="directed",
                                  view=view)
    pg.four_clique_count(view, pg.make_provider("bf_and", sketched=dsk))
ex = pg.make_provider("exact_merge", view=view)
pg.triangle_count(view, ex)
pg.four_clique_count(view, ex)
pg.four_clique_count(view, pg.make_provider("exact_merge", graph=g))
for cap in ("512", "4"):
    os.environ["PG_C4S_CAP"] = cap
    for kind in ("khash", "onehash", "kmv"):
        dsk = pg.build_sketched_graph(g, kind, s=1.0, k_override=16, source="directed", view=view)
        pg.four_clique_count(view, pg.make_provider(kind, sketched=dsk))
os.environ.pop("PG_C4S_CAP")

# generators, link prediction
pg.generate_chung_lu(1 << 12, 16, 2.1, 3)
pg.generate_erdos_renyi_gnm(4096, 30000, 0)
gs = pg.generate_kronecker(10, 8, 3)
split = pg.make_link_prediction_split(gs, 0.1, 0)
skl = pg.build_sketched_graph(split.sparse_graph, "bloom", s=1.0, b=2, bits_override=1024)
for measure in ("jaccard", "adamic_adar"):
    prov = pg.make_provider("bf_and" if measure == "jaccard" else "exact_merge",
                            **({"sketched": skl} if measure == "jaccard" else {"graph": split.sparse_graph}))
    pg.link_prediction_eval(gs, split, measure, prov, 100)
print("sanitize cases ok")
