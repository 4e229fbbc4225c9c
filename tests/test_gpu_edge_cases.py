"""Degenerate inputs through every entry point on the device: the empty
graph, an edgeless graph, a single edge, empty query batches, degrees below
and above k.  Values are checked against the oracle or the obvious answer."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KINDS = [("bloom", "bf_and", {"b": 2, "bits_override": 256}),
         ("bloom", "bf_or", {"b": 1, "bits_override": 576}),
         ("khash", "khash", {"k_override": 8}),
         ("onehash", "onehash", {"k_override": 32}),
         ("kmv", "kmv", {"k_override": 32})]


@pytest.fixture(scope="module")
def pg():
    import paper_2208_11469_b200 as pg
    return pg


def _graphs(pg):
    return {
        "empty": pg.CsrGraph(np.zeros(1, np.int64), np.empty(0, np.int64)),
        "edgeless": pg.CsrGraph(np.zeros(7, np.int64), np.empty(0, np.int64)),
        "one_edge": pg.CsrGraph.from_edges([[2, 5]], 6),
        "triangle_plus": pg.CsrGraph.from_edges([[0, 1], [1, 2], [0, 2], [2, 3], [3, 4]], 8),
    }


@pytest.mark.parametrize("sk_kind,kind,kw", KINDS)
def test_degenerate_graphs_all_kinds(pg, sk_kind, kind, kw):
    for name, g in _graphs(pg).items():
        sk = pg.build_sketched_graph(g, sk_kind, s=1.0, **kw)
        assert sk.n == g.n
        est = pg.tc_estimate(g, sk, kind)
        if g.m == 0:
            assert est == 0.0, name
        p = pg.make_provider(kind, sketched=sk)
        assert len(p.pair_many(np.empty(0, np.int64), np.empty(0, np.int64))) == 0
        if g.m:
            e = g.edges()
            assert np.all(np.isfinite(p.pair_many(e[:, 0], e[:, 1])))
        jp = pg.jarvis_patrick_cluster(g, p, 0.5)
        assert jp.singleton_count + len(np.unique(jp.kept_edges)) == g.n
        if sk_kind == "khash":
            jc = pg.jaccard_cluster_count(g, sk, 0.1)
            assert int(jc.match_hist.sum()) == g.m


def test_degenerate_exact_and_4clique(pg):
    for name, g in _graphs(pg).items():
        view = pg.degree_order(g)
        ex = pg.make_provider("exact_merge", view=view)
        tc = pg.triangle_count(view, ex)
        assert tc == (1 if name == "triangle_plus" else 0), name
        assert pg.four_clique_count(view, ex) == 0
        dsk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=512,
                                      source="directed", view=view)
        bp = pg.make_provider("bf_and", sketched=dsk)
        c4 = pg.four_clique_count(view, bp)
        assert np.isfinite(c4)
        assert pg.tc_estimate(g, kind="exact_merge") == float(tc)


def test_degenerate_link_prediction_and_baselines(pg):
    for name, g in _graphs(pg).items():
        split = pg.make_link_prediction_split(g, 0.5, 1)
        ex = pg.make_provider("exact_merge", graph=split.sparse_graph)
        assert pg.link_prediction_eval(g, split, "jaccard", ex, 10) >= 0
        if g.n:
            assert pg.doulion_tc(g, 1.0, 0) == (1.0 if name == "triangle_plus" else 0.0)
            view = pg.degree_order(g)
            assert pg.reduced_execution_tc(view, 1.0, 0) == \
                (1.0 if name == "triangle_plus" else 0.0)


def test_degree_below_and_above_k(pg):
    from oracle import oracle as O
    # star + path: degrees 1..40 around k = 16
    edges = [[0, i] for i in range(1, 41)] + [[i, i + 1] for i in range(1, 40)]
    g = pg.CsrGraph.from_edges(edges)
    for sk_kind, k in (("khash", 16), ("onehash", 16), ("kmv", 16)):
        sk = pg.build_sketched_graph(g, sk_kind, s=1.0, k_override=k)
        if sk_kind == "khash":
            assert np.array_equal(sk.entries, O.C.build_khash(g.offsets, g.adjacency, k))
        elif sk_kind == "onehash":
            ent, ln = O.C.build_onehash(g.offsets, g.adjacency, k)
            assert np.array_equal(sk.entries, ent) and np.array_equal(sk.lengths, ln)
        else:
            val, ln = O.C.build_kmv(g.offsets, g.adjacency, k)
            assert np.array_equal(sk.values, val) and np.array_equal(sk.lengths, ln)
