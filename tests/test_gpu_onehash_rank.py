"""1-Hash hash-rank rows (pg_hash_rank_table, pg_onehash_rank_rows) and the
per-warp-table TC engine over them (pg_tc_minhash with onehash = 2).

The rank rows relabel the stored IDs by the position of their h0 word among
all vertices (exact: h0 is a bijection), sorted ascending, so the engine can
stop probing v's row at u's largest rank.  Checked: the table and the rows
against a numpy restatement (hashing.py:114-118 hash_words); the fused pass
over rank rows against the same pass over ID rows (identical integers) and
against the reference-pinned tc_estimate.
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

INT32_MAX = np.iinfo(np.int32).max
DEFAULT_HASH_SEED = 0x9E3779B97F4A7C15


@pytest.fixture(scope="module")
def pg():
    import paper_2208_11469_b200 as pg
    return pg


@pytest.mark.parametrize("n", [1, 2, 33, 5000, 70001])
def test_hash_rank_table(pg, n):
    import torch
    from paper_2208_11469_b200 import _native as N
    seeds = O.C.seeds(DEFAULT_HASH_SEED, 1)
    sd = torch.from_numpy(seeds.view(np.int64)).cuda()
    rank_of = torch.empty(n, dtype=torch.int32, device="cuda")
    N.call("pg_hash_rank_table", n, N.ptr(sd), N.ptr(rank_of), N.stream_handle())
    w = O.NumpyPort._hash(int(seeds[0]), np.arange(n, dtype=np.int64))
    want = np.empty(n, dtype=np.int64)
    want[np.argsort(w, kind="stable")] = np.arange(n)
    assert np.array_equal(rank_of.cpu().numpy(), want)


@pytest.mark.parametrize("k", [32, 64, 128])
def test_rank_rows(pg, k):
    g = pg.generate_kronecker(12, 16, 3)
    sk = pg.build_sketched_graph(g, "onehash", s=1.0, k_override=k)
    p = pg.make_provider("onehash", sketched=sk)
    rows = p._rank_rows().cpu().numpy()
    seeds = O.C.seeds(DEFAULT_HASH_SEED, 1)
    w = O.NumpyPort._hash(int(seeds[0]), np.arange(g.n, dtype=np.int64))
    rank = np.empty(g.n, dtype=np.int64)
    rank[np.argsort(w, kind="stable")] = np.arange(g.n)
    ent = sk.entries
    want = np.where(ent >= 0, rank[np.maximum(ent, 0)], INT32_MAX)
    want.sort(axis=1)
    # stored interleaved over the engine's lanes per row
    from paper_2208_11469_b200 import _native as N
    group = 32 // N.onehash_block_pad(k)
    j = np.arange(k)
    slot = (j % group) * (k // group) + j // group
    inter = np.empty_like(want)
    inter[:, slot] = want
    assert np.array_equal(rows, inter)


@pytest.mark.parametrize("graph", ["rmat12", "rmat15", "er", "star"])
@pytest.mark.parametrize("k", [32, 64, 128])
@pytest.mark.parametrize("orient,layout", [("degree", "sorted"), ("id", "sorted"), ("degree", "plain")])
def test_tc_rank_rows_equal_id_rows(pg, monkeypatch, graph, k, orient, layout):
    from paper_2208_11469_b200.mining import tc_counts
    monkeypatch.setenv("PG_TC_ORIENT", orient)
    monkeypatch.setenv("PG_ONEHASH_LAYOUT", layout)
    if graph == "rmat12":
        g = pg.generate_kronecker(12, 16, 9)
    elif graph == "rmat15":
        g = pg.generate_kronecker(15, 16, 10)
    elif graph == "er":
        g = pg.generate_erdos_renyi_gnm(3000, 60000, 4)
    else:
        e = [[0, i] for i in range(1, 500)] + [[i, i + 1] for i in range(1, 499)]
        e += [[i, j] for i in range(1, 50) for j in range(i + 1, 50)]
        g = pg.CsrGraph.from_edges(e, 500)
    sk = pg.build_sketched_graph(g, "onehash", s=1.0, k_override=k)
    p = pg.make_provider("onehash", sketched=sk)
    assert p._rank_rows() is not None
    lay = p._tc_layout(g.device())
    assert lay.kind == (orient + "+onehash-rank" if layout == "sorted" else "id")
    assert int((lay.vs >= 0).sum().item()) == g.m
    got = tc_counts(p, g.device()).cpu().numpy()
    # two shards add up to the whole (padded ranges split on 32-slot units)
    parts = tc_counts(p, g.device(), 0, 2).cpu().numpy() + tc_counts(p, g.device(), 1, 2).cpu().numpy()
    assert np.array_equal(parts, got)
    monkeypatch.setenv("PG_ONEHASH_ROWS", "id")
    p2 = pg.make_provider("onehash", sketched=sk)
    assert p2._rank_rows() is None
    want = tc_counts(p2, g.device()).cpu().numpy()
    assert np.array_equal(got, want)
    # and the per-edge reference semantics (providers.py:197-232) through the oracle
    e = g.edges()
    m = O.C.pairs_minhash(sk.entries, k, True, e[:, 0], e[:, 1])
    hist = np.bincount(m, minlength=k + 1)
    sz = np.diff(g.offsets)
    verb = (sz[e[:, 0]] <= k) & (sz[e[:, 1]] <= k)
    assert np.array_equal(got[:k + 1], np.bincount(m[~verb], minlength=k + 1))
    assert int(got[-1]) == int(m[verb].sum())
    assert hist.sum() == g.m


@pytest.mark.parametrize("graph", ["rmat12", "hub6000"])
def test_in_lists_and_sorted_rows(pg, graph):
    """pg_degree_in_lists = the transpose of degree_order's N+ lists;
    pg_onehash_sort_rows = every row stably counting-sorted by
    ceil(pg_onehash_prefix_counts / group)."""
    import torch
    from paper_2208_11469_b200 import _native as N
    k = 64
    if graph == "rmat12":
        g = pg.generate_kronecker(12, 16, 11)
    else:  # rows above 2,048 entries take the CTA-per-row sort
        rng = np.random.default_rng(5)
        e = [[0, i] for i in range(1, 6001)] + [[1, i] for i in range(2, 3001)]
        e += [[int(a), int(b)] for a, b in rng.integers(2, 6001, size=(40000, 2)) if a != b]
        g = pg.CsrGraph.from_edges(e, 6100)
    dev = g.device()
    rank = dev.degree_rank()[0]
    half = dev.nnz // 2
    off = torch.empty(g.n + 1, dtype=torch.int64, device="cuda")
    adj = torch.empty(half, dtype=torch.int32, device="cuda")
    N.call("pg_degree_in_lists", N.ptr(dev.offsets), N.ptr(dev.adj), g.n, dev.nnz, N.ptr(rank),
           N.ptr(off), N.ptr(adj), N.stream_handle())
    hr = rank.cpu().numpy()
    src = np.repeat(np.arange(g.n), np.diff(g.offsets))
    keep = hr[g.adjacency] < hr[src]
    assert np.array_equal(adj.cpu().numpy(), g.adjacency[keep])
    want_off = np.concatenate([[0], np.cumsum(np.bincount(src[keep], minlength=g.n))])
    assert np.array_equal(off.cpu().numpy(), want_off)
    # rows sorted by probe-register count
    sk = pg.build_sketched_graph(g, "onehash", s=1.0, k_override=k)
    p = pg.make_provider("onehash", sketched=sk)
    rows = p._rank_rows()
    d = sk.device_tensors()
    group = 32 // N.onehash_block_pad(k)
    out = torch.empty_like(adj)
    N.call("pg_onehash_sort_rows", N.ptr(off), N.ptr(adj), g.n, N.ptr(rows), N.ptr(d["lengths"]), k, group,
           N.ptr(out), N.stream_handle())
    ts = torch.from_numpy(src[keep].astype(np.int32)).cuda()
    bp = torch.empty(half, dtype=torch.int32, device="cuda")
    N.call("pg_onehash_prefix_counts", N.ptr(rows), N.ptr(d["lengths"]), k, group, N.ptr(ts), N.ptr(adj),
           half, N.ptr(bp), N.stream_handle())
    bucket = (bp.cpu().numpy() + group - 1) // group
    a, o = adj.cpu().numpy(), out.cpu().numpy()
    t = src[keep]
    order = np.lexsort((np.arange(half), bucket, t))  # stable by (row, bucket)
    assert np.array_equal(o, a[order])


def test_rank_rows_bad_arguments(pg):
    from paper_2208_11469_b200 import _native as N
    from paper_2208_11469_b200.providers import UnsupportedCombinationError
    with pytest.raises(UnsupportedCombinationError):
        N.call("pg_onehash_rank_rows", None, 5, 48, None, 8, None, None)
    with pytest.raises(UnsupportedCombinationError):  # rank rows need the padded layout
        N.call("pg_tc_minhash", None, 64, 2, None, None, None, 0, 0, 0, 1, 1, 1, None)
