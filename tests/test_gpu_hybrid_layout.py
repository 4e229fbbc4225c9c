"""DeviceCsr.hybrid_slots: the degree-oriented group-u slot layout with the
short N+ rows regrouped by their higher-rank endpoint.  Every undirected edge
must appear exactly once, every slot group must share its u, and the fused
Bloom pass over it must give the histogram of the plain layouts (the per-edge
popcount of providers.py:150-162 is symmetric in (u, v))."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    import paper_2208_11469_b200 as pg
    return pg


@pytest.mark.parametrize("base", ["degree", "id"])
@pytest.mark.parametrize("graph", ["rmat12", "rmat14", "er", "star"])
@pytest.mark.parametrize("thr", [1, 2, 4, 8])
def test_hybrid_slots_cover_every_edge_once(pg, graph, thr, base):
    if graph == "rmat12":
        g = pg.generate_kronecker(12, 16, 3)
    elif graph == "rmat14":
        g = pg.generate_kronecker(14, 8, 5)
    elif graph == "er":
        g = pg.generate_erdos_renyi_gnm(2000, 9000, 2)
    else:
        e = [[0, i] for i in range(1, 300)] + [[i, i + 1] for i in range(1, 299)]
        g = pg.CsrGraph.from_edges(e, 320)
    dev = g.device()
    pad = 8
    ug, vs, slots = dev.hybrid_slots(pad, thr, base)
    ug, vs = ug.cpu().numpy(), vs.cpu().numpy()
    assert slots % pad == 0 and len(vs) == slots and len(ug) == slots // pad
    us = np.repeat(ug, pad)
    real = vs >= 0
    assert int(real.sum()) == g.m
    a, b = np.minimum(us[real], vs[real]).astype(np.int64), np.maximum(us[real], vs[real]).astype(np.int64)
    got = np.sort(a * g.n + b)
    e = g.edges()
    assert np.array_equal(got, np.sort(e[:, 0] * g.n + e[:, 1]))
    # what it is for: fewer pad slots on skewed graphs
    if graph.startswith("rmat") and thr < pad:
        plain = dev.hub_slots(pad, 0)[2] if base == "degree" else dev.upper_edges_group_u(pad)[2]
        assert slots < plain


def test_bloom_tc_over_id_hybrid_layout(pg, monkeypatch):
    from paper_2208_11469_b200.mining import tc_counts
    g = pg.generate_kronecker(13, 16, 7)
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=1024)
    monkeypatch.setenv("PG_TC_ORIENT", "id")
    want = tc_counts(pg.make_provider("bf_and", sketched=sk), g.device()).cpu().numpy()
    monkeypatch.setenv("PG_TC_HYBRID_ID", "2")
    p = pg.make_provider("bf_and", sketched=sk)
    assert p._tc_layout(g.device()).regroup == 2
    assert np.array_equal(tc_counts(p, g.device()).cpu().numpy(), want)


@pytest.mark.parametrize("thr", ["0", "2", "5"])
def test_bloom_tc_over_hybrid_layout(pg, monkeypatch, thr):
    from paper_2208_11469_b200.mining import tc_counts
    g = pg.generate_kronecker(13, 16, 7)
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048)
    monkeypatch.setenv("PG_TC_ORIENT", "id")
    want = tc_counts(pg.make_provider("bf_and", sketched=sk), g.device()).cpu().numpy()
    monkeypatch.setenv("PG_TC_ORIENT", "degree")
    monkeypatch.setenv("PG_TC_HYBRID", thr)
    p = pg.make_provider("bf_and", sketched=sk)
    got = tc_counts(p, g.device()).cpu().numpy()
    assert np.array_equal(got, want)
    parts = sum(tc_counts(p, g.device(), r, 3).cpu().numpy() for r in range(3))
    assert np.array_equal(parts, want)
