"""Link prediction on the device against the reference
(tests/golden/linkpred.json from make_golden_linkpred.py): the split, the
two-hop candidates, every candidate's vertex_similarity score (bit-exact,
as a checksum of the float64 bytes) and link_prediction_eval hit counts."""

import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLD = json.load(open(os.path.join(HERE, "linkpred.json")))
TOPS = [1, 10, 100, 1000, 10 ** 9]
PROVIDERS = {
    "exact": (None, {}, "exact_merge"),
    "bf_and": ("bloom", {"b": 2, "bits_override": 256}, "bf_and"),
    "bf_or": ("bloom", {"b": 2, "bits_override": 256}, "bf_or"),
    "khash": ("khash", {"k_override": 16}, "khash"),
    "onehash": ("onehash", {"k_override": 16}, "onehash"),
    "kmv": ("kmv", {"k_override": 16}, "kmv"),
}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _graph(pg, name):
    if name == "rmat8":
        return pg.generate_kronecker(8, 8, 21)
    return pg.generate_erdos_renyi_gnm(300, 1500, 6)


@pytest.mark.parametrize("case", sorted(GOLD))
def test_linkpred_matches_reference(case):
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import mining as M
    rec = GOLD[case]
    g = _graph(pg, case)
    assert (g.n, g.m) == (rec["n"], rec["m"])
    split = pg.make_link_prediction_split(g, rec["fraction"], rec["seed"])
    sp = split.sparse_graph
    assert sha(split.edges_removed.astype("<i8")) == rec["edges_removed"]
    assert sha(sp.adjacency.astype("<i8")) == rec["sparse_adjacency"]
    cands = M._two_hop_candidates(sp)
    assert len(cands) == rec["candidate_count"]
    assert sha(cands.astype("<i8")) == rec["candidates"]
    keys = M._two_hop_keys(sp)
    for pname, (skind, kw, ekind) in PROVIDERS.items():
        if skind is None:
            prov = pg.make_provider(ekind, graph=sp)
        else:
            sk = pg.build_sketched_graph(sp, skind, s=1.0, seed=rec["seed"] + 1000, **kw)
            prov = pg.make_provider(ekind, sketched=sk)
        for meas in ("jaccard", "overlap", "common_neighbors", "total_neighbors",
                     "adamic_adar", "resource_allocation"):
            want = rec["results"][f"{pname}/{meas}"]
            if "error" in want:
                with pytest.raises(Exception) as ei:
                    M.similarity_scores(sp, keys, meas, prov)
                assert type(ei.value).__name__ == want["error"]
                with pytest.raises(Exception):
                    pg.link_prediction_eval(g, split, meas, prov, 10)
                continue
            sc = M.similarity_scores(sp, keys, meas, prov).cpu().numpy()
            assert sha(sc.astype("<f8")) == want["scores"], (pname, meas)
            hits = [pg.link_prediction_eval(g, split, meas, prov, t) for t in TOPS]
            assert hits == want["hits"], (pname, meas)


def test_linkpred_edge_cases():
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import mining as M
    g = pg.CsrGraph.from_edges([[0, 1], [1, 2], [3, 4]], 6)
    assert M._two_hop_candidates(g).tolist() == [[0, 2]]
    split = pg.make_link_prediction_split(g, 0.0, 1)
    ex = pg.make_provider("exact_merge", graph=split.sparse_graph)
    assert pg.link_prediction_eval(g, split, "jaccard", ex, 0) == 0
    assert pg.link_prediction_eval(g, split, "jaccard", ex, 5) == 0
    with pytest.raises(ValueError):
        pg.make_link_prediction_split(g, 1.5, 0)
    bad = pg.mining.LinkPredSplit(split.sparse_graph, split.edges_sparse[:1],
                                  split.edges_removed, 0.0, 1)
    with pytest.raises(ValueError):
        pg.link_prediction_eval(g, bad, "jaccard", ex, 5)
    # a triangle has no non-adjacent two-hop pairs
    tri = pg.CsrGraph.from_edges([[0, 1], [1, 2], [0, 2]])
    assert len(M._two_hop_candidates(tri)) == 0
