"""Jarvis-Patrick on the device (pg_jp_components) against the reference's
host union-find semantics (mining.py:213-245), restated here with scipy."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _host_jp(graph, scores, tau):
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    e = graph.edges()
    kept = e[scores > tau]
    touched = np.unique(kept.reshape(-1))
    if len(kept):
        a = coo_matrix((np.ones(len(kept)), (kept[:, 0], kept[:, 1])), shape=(graph.n, graph.n))
        _, labels = connected_components(a, directed=False)
        clusters = len(np.unique(labels[touched]))
    else:
        clusters = 0
    return kept, clusters, graph.n - len(touched)


@pytest.mark.parametrize("kind,sk_kind", [("bf_and", "bloom"), ("khash", "khash"),
                                          ("exact_merge", None)])
def test_jp_matches_host_union_find(kind, sk_kind):
    import paper_2208_11469_b200 as pg
    g = pg.generate_kronecker(15, 8, 5)
    if sk_kind:
        sk = pg.build_sketched_graph(g, sk_kind, s=1.0, b=2, bits_override=512, k_override=32)
        p = pg.make_provider(kind, sketched=sk)
    else:
        p = pg.make_provider(kind, graph=g)
    e = g.edges()
    scores = np.asarray(p.pair_many(e[:, 0], e[:, 1]), dtype=np.float64)
    for tau in (-1.0, 0.0, 0.5, 1.0, 2.0, 5.0, float(scores.max()), 1e18):
        got = pg.jarvis_patrick_cluster(g, p, tau)
        kept, clusters, singles = _host_jp(g, scores, tau)
        assert np.array_equal(got.kept_edges, kept), tau
        assert got.cluster_count == clusters, tau
        assert got.singleton_count == singles, tau


def test_jp_components_long_chains():
    """A path and a star stress the union-find's hooking and path splitting
    (all edges kept)."""
    import torch
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import _native as N
    n = 200_003
    path = np.stack([np.arange(0, 100_000), np.arange(1, 100_001)], 1)
    star = np.stack([np.full(99_000, 100_002), np.arange(101_003, 200_003)], 1)
    e = np.concatenate([path, star]).astype(np.int32)
    rng = np.random.default_rng(3)
    e = e[rng.permutation(len(e))]  # random union order
    us = torch.from_numpy(np.ascontiguousarray(e[:, 0])).cuda()
    vs = torch.from_numpy(np.ascontiguousarray(e[:, 1])).cuda()
    scores = torch.ones(len(e), dtype=torch.float64, device="cuda")
    out = torch.empty(3, dtype=torch.int64, device="cuda")
    N.call("pg_jp_components", N.ptr(us), N.ptr(vs), N.ptr(scores), len(e), 0.5, n,
           None, N.ptr(out), N.stream_handle())
    kept, clusters, touched = out.cpu().tolist()
    assert kept == len(e)
    assert clusters == 2
    assert touched == 100_001 + 99_001
    del pg
