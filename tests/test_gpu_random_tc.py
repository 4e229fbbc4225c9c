"""Randomised end-to-end check of every fused TC engine (Bloom wide / group-u,
k-Hash wide, 1-Hash per-warp table, KMV rank directory) against the C
oracle's per-edge restatement of the reference (providers.py:137-301) on
seeded random graphs: ER plus planted hubs, isolated vertices and long
paths, at every sketch width the engines dispatch on."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

RTOL = 1e-12


@pytest.fixture(scope="module")
def pg():
    import paper_2208_11469_b200 as pg
    return pg


def _graph(pg, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(50, 3000))
    m = int(rng.integers(n, 12 * n))
    e = rng.integers(0, n, size=(m, 2))
    hubs = rng.choice(n, size=min(3, n), replace=False)
    for h in hubs:  # planted hubs: rows far longer than any k
        nb = rng.choice(n, size=min(n - 1, int(rng.integers(100, 1500))), replace=False)
        e = np.concatenate([e, np.stack([np.full(len(nb), h), nb], 1)])
    path = np.arange(n - 40, n - 1)
    e = np.concatenate([e, np.stack([path, path + 1], 1)])
    e = e[e[:, 0] != e[:, 1]]
    return pg.CsrGraph.from_edges(e, n + 5)  # + isolated vertices


def _oracle_tc(kind, g, sk, k=None, bits=None, b=None):
    e = g.edges()
    sz = np.diff(g.offsets)
    if kind == "bloom":
        pop = O.C.pairs_bloom(sk.bit_matrix, bits, False, e[:, 0], e[:, 1])
        return float(np.sum(O.bloom_edge_estimates(pop, "bf_and", bits, b))) / 3.0
    if kind in ("khash", "onehash"):
        m = O.C.pairs_minhash(sk.entries, k, kind == "onehash", e[:, 0], e[:, 1])
        return float(np.sum(O.minhash_edge_estimates(m, k, sz[e[:, 0]], sz[e[:, 1]],
                                                     kind == "onehash"))) / 3.0
    _, _, est = O.C.pairs_kmv(sk.values, sk.lengths, k, sz, e[:, 0], e[:, 1])
    return float(np.sum(est)) / 3.0


@pytest.mark.parametrize("seed", range(8))
def test_random_graphs_all_engines(pg, seed):
    g = _graph(pg, seed)
    cases = [("bloom", dict(bits_override=512, b=1)), ("bloom", dict(bits_override=1024, b=2)),
             ("bloom", dict(bits_override=2048, b=3)), ("khash", dict(k_override=32)),
             ("khash", dict(k_override=64)), ("onehash", dict(k_override=32)),
             ("onehash", dict(k_override=64)), ("onehash", dict(k_override=128)),
             ("kmv", dict(k_override=32)), ("kmv", dict(k_override=64)), ("kmv", dict(k_override=128))]
    for kind, kw in cases:
        sk = pg.build_sketched_graph(g, kind, s=1.0, seed=1000 + seed, **kw)
        # the builders against the C oracle's builders (same seed family)
        if kind == "bloom":
            rows, ones = O.C.build_bloom(g.offsets, g.adjacency, kw["bits_override"], kw["b"], seed=1000 + seed)
            assert np.array_equal(sk.bit_matrix, rows) and np.array_equal(sk.ones, ones)
        elif kind == "khash":
            assert np.array_equal(sk.entries, O.C.build_khash(g.offsets, g.adjacency, kw["k_override"],
                                                              seed=1000 + seed))
        elif kind == "onehash":
            ent, ln = O.C.build_onehash(g.offsets, g.adjacency, kw["k_override"], seed=1000 + seed)
            assert np.array_equal(sk.entries, ent) and np.array_equal(sk.lengths, ln)
        else:
            val, ln = O.C.build_kmv(g.offsets, g.adjacency, kw["k_override"], seed=1000 + seed)
            assert np.array_equal(sk.values, val) and np.array_equal(sk.lengths, ln)
        est_kind = "bf_and" if kind == "bloom" else kind
        got = pg.tc_estimate(g, sk, est_kind)
        want = _oracle_tc(kind, g, sk, k=kw.get("k_override"), bits=kw.get("bits_override"), b=kw.get("b"))
        assert got == pytest.approx(want, rel=RTOL, abs=1e-9), (seed, kind, kw)
