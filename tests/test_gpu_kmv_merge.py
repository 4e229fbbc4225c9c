"""KMV thread-per-edge merge engine (pg_tc_kmv_merge, pg_kmv_merge_partition)
against the reference semantics (providers.py:266-301 KmvProvider.pair_many).

One lane per edge slot merges the two rank rows with two pointers and stops
after k_eff steps where only the k_eff-th distinct union value is needed.
Checked here: whole-graph sums for both edge orientations, with and without
the [short | full] partition, against the C oracle's restatement and the
values engine; crafted rank rows (dense clusters, short and empty rows,
verbatim and degenerate k_eff cases, shared elements, pad slots) edge by edge;
the partition itself (stable, exact split); run-to-run bit identity.
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

RTOL_SUM = 1e-12
INT32_MAX = np.iinfo(np.int32).max


@pytest.fixture(scope="module")
def pg():
    import paper_2208_11469_b200 as pg
    return pg


def _graph(pg, graph):
    if graph == "rmat11":
        return pg.generate_kronecker(11, 16, 7)
    if graph == "rmat13":
        return pg.generate_kronecker(13, 8, 8)
    if graph == "star":  # one hub over two cliques of small vertices
        e = [[0, i] for i in range(1, 400)]
        e += [[i, j] for i in range(1, 40) for j in range(i + 1, 40)]
        e += [[i, i + 1] for i in range(40, 399)]
        return pg.CsrGraph.from_edges(e, 400)
    return pg.generate_erdos_renyi_gnm(3000, 60000, 4)


@pytest.mark.parametrize("graph", ["rmat11", "rmat13", "star", "er"])
@pytest.mark.parametrize("k", [32, 64, 128])
@pytest.mark.parametrize("orient,part", [("degree", "1"), ("id", "1"), ("degree", "0")])
def test_merge_tc_vs_oracle(pg, monkeypatch, graph, k, orient, part):
    from paper_2208_11469_b200.mining import tc_counts
    monkeypatch.setenv("PG_TC_ORIENT", orient)
    monkeypatch.setenv("PG_KMV_PARTITION", part)
    g = _graph(pg, graph)
    sk = pg.build_sketched_graph(g, "kmv", s=1.0, k_override=k)
    p = pg.make_provider("kmv", sketched=sk)
    assert p._merge_engine()
    lay = p._tc_layout(g.device())
    assert lay.kind == orient + "+kmv-merge" and lay.slots == g.m
    got = p._tc_combine(tc_counts(p, g.device()).cpu().numpy())
    again = p._tc_combine(tc_counts(p, g.device()).cpu().numpy())
    e = g.edges()
    _, _, est = O.C.pairs_kmv(sk.values, sk.lengths, k, np.diff(g.offsets), e[:, 0], e[:, 1])
    want = float(np.sum(est))
    assert got == pytest.approx(want, rel=RTOL_SUM, abs=1e-9)
    assert got == again  # fixed-slot partials, fixed-order sum
    assert pg.tc_estimate(g, sk, "kmv") == pytest.approx(want / 3.0, rel=RTOL_SUM, abs=1e-9)
    # the rank-directory engine over the same sketches
    monkeypatch.setenv("PG_KMV_ENGINE", "ranked")
    sk._kmv_merge_layout = None
    p2 = pg.make_provider("kmv", sketched=sk)
    assert not p2._merge_engine()
    ranked = p2._tc_combine(tc_counts(p2, g.device()).cpu().numpy())
    assert ranked == pytest.approx(want, rel=RTOL_SUM, abs=1e-9)


@pytest.mark.parametrize("k", [32, 64, 128])
def test_merge_tc_s16_vs_values_engine(pg, k):
    """R-MAT s16 (1.0 M edges, hubs of degree > 10^4): the merge engine over
    rank rows against the values engine (pg_tc_kmv) over the same sketches,
    whole graph and two shard ranges."""
    import torch
    from paper_2208_11469_b200 import _native as N
    g = pg.generate_kronecker(16, 16, 5)
    sk = pg.build_sketched_graph(g, "kmv", s=1.0, k_override=k)
    p = pg.make_provider("kmv", sketched=sk)
    lay = p._tc_layout(g.device())
    d = sk.device_tensors()
    out = torch.empty(1, dtype=torch.float64, device="cuda")

    def values(us, vs, b, e):
        N.call("pg_tc_kmv", N.ptr(d["values"]), N.ptr(d["lengths"]), k, N.ptr(d["sizes"]),
               N.ptr(us), N.ptr(vs), b, e, N.ptr(out), N.stream_handle())
        return float(out.item())

    def merge(b, e):
        return float(p._tc_counts(lay.us, lay.vs, b, e, lay.padded).item())

    whole = values(lay.us, lay.vs, 0, lay.slots)
    assert merge(0, lay.slots) == pytest.approx(whole, rel=RTOL_SUM)
    cut = lay.slots // 3 + 5
    assert merge(0, cut) + merge(cut, lay.slots) == pytest.approx(whole, rel=RTOL_SUM)
    assert merge(cut, lay.slots) == pytest.approx(values(lay.us, lay.vs, cut, lay.slots), rel=RTOL_SUM)
    assert merge(7, 7) == 0.0


def _crafted(k, n_rows, rng):
    pool_hi = 50_000
    rows = np.full((n_rows, k), INT32_MAX, dtype=np.int64)
    lens = np.zeros(n_rows, dtype=np.int64)
    shared = np.sort(rng.choice(pool_hi, size=3 * k, replace=False))
    for r in range(n_rows):
        kind = r % 7
        if kind == 0:    # spread, overlapping the shared pool
            pick = np.concatenate([rng.choice(shared, k // 2, replace=False),
                                   rng.choice(pool_hi, k, replace=False)])
        elif kind == 1:  # dense cluster
            base = int(rng.integers(0, pool_hi - 4 * k))
            pick = np.concatenate([base + rng.choice(2 * k, (3 * k) // 4, replace=False),
                                   rng.choice(pool_hi, k, replace=False)])
        elif kind == 2:  # consecutive ranks
            base = int(rng.integers(0, pool_hi - k))
            pick = base + np.arange(k)
        elif kind == 3:  # short row
            pick = rng.choice(shared, int(rng.integers(1, 5)), replace=False)
        elif kind == 4:  # empty row
            pick = np.empty(0, dtype=np.int64)
        elif kind == 5:  # a full row of shared elements only (many common values)
            pick = shared[:k] if r % 2 else shared[k // 2:k // 2 + k]
        else:            # k/2 elements
            pick = rng.choice(pool_hi, k // 2, replace=False)
        pick = np.unique(pick)[:k]
        rows[r, :len(pick)] = pick
        lens[r] = len(pick)
    return rows, lens


@pytest.mark.parametrize("k", [32, 64, 128])
def test_merge_crafted_rows_edge_by_edge(pg, k):
    import torch
    from paper_2208_11469_b200 import _native as N
    rng = np.random.default_rng(100 + k)
    n_rows = 49
    ranks, lens = _crafted(k, n_rows, rng)
    rank_values = np.cumsum(rng.random(60_000) ** 3 + 1e-9) * 1e-5
    vals = np.where(ranks == INT32_MAX, np.inf, rank_values[np.minimum(ranks, 59_999)])
    sizes = np.where(np.arange(n_rows) % 3 == 0, lens,
                     lens + rng.integers(1, 10 * k, n_rows)).astype(np.int64)
    pairs = np.array([(u, v) for u in range(n_rows) for v in range(n_rows) if u != v])
    # every other slot is a pad (u, -1)
    us = np.repeat(pairs[:, 0], 2).astype(np.int32)
    vs = np.full(len(pairs) * 2, -1, dtype=np.int32)
    vs[::2] = pairs[:, 1]
    dev = {name: torch.from_numpy(np.ascontiguousarray(a)).cuda() for name, a in (
        ("ranks", ranks.astype(np.int32)), ("rv", rank_values), ("lens", lens.astype(np.int32)),
        ("sizes", sizes.astype(np.int32)), ("us", us), ("vs", vs))}
    out = torch.empty(1, dtype=torch.float64, device="cuda")

    def run(b, e, uk="us", vk="vs"):
        N.call("pg_tc_kmv_merge", N.ptr(dev["ranks"]), N.ptr(dev["rv"]), N.ptr(dev["lens"]), k,
               N.ptr(dev["sizes"]), N.ptr(dev[uk]), N.ptr(dev[vk]), b, e, N.ptr(out),
               N.stream_handle())
        return float(out.item())

    _, _, est = O.C.pairs_kmv(vals, lens, k, sizes, pairs[:, 0], pairs[:, 1])
    total = float(np.sum(est))
    assert run(0, len(us)) == pytest.approx(total, rel=RTOL_SUM)
    for i in rng.choice(len(pairs), 150, replace=False):
        assert run(2 * int(i), 2 * int(i) + 2) == est[i], (pairs[i], lens[pairs[i]], sizes[pairs[i]])
    # 32-slot blocks starting anywhere (lanes of one warp in every branch at once)
    for b in rng.integers(0, len(us) - 70, 20):
        b = int(b)
        want = float(np.sum(est[(b + 1) // 2:(b + 64 + 1) // 2]))
        assert run(b, b + 64) == pytest.approx(want, rel=1e-13)
    # the partitioned order gives the same sum
    pu, pv = torch.empty_like(dev["us"]), torch.empty_like(dev["vs"])
    import ctypes
    split = ctypes.c_int64()
    N.call("pg_kmv_merge_partition", N.ptr(dev["us"]), N.ptr(dev["vs"]), len(us), N.ptr(dev["sizes"]),
           N.ptr(dev["lens"]), k, 1, N.ptr(pu), N.ptr(pv), ctypes.byref(split), N.stream_handle())
    dev["pu"], dev["pv"] = pu, pv
    assert run(0, len(us), "pu", "pv") == pytest.approx(total, rel=RTOL_SUM)
    # the partition: stable, short merges first
    hu, hv = pu.cpu().numpy(), pv.cpu().numpy()
    su_, sv_ = sizes[us], sizes[np.maximum(vs, 0)]
    short = (vs >= 0) & ~((su_ <= k) & (sv_ <= k)) & (np.minimum(lens[us], lens[np.maximum(vs, 0)]) >= 2)
    assert split.value == int(short.sum())
    assert np.array_equal(hu[:split.value], us[short]) and np.array_equal(hv[:split.value], vs[short])
    assert np.array_equal(hu[split.value:], us[~short]) and np.array_equal(hv[split.value:], vs[~short])


@pytest.mark.parametrize("buckets", [1, 4, 8])
@pytest.mark.parametrize("count", [1, 31, 2048, 2049, 100_003])
def test_partition_sizes(pg, count, buckets):
    import ctypes
    import torch
    from paper_2208_11469_b200 import _native as N
    rng = np.random.default_rng(count)
    n, k = 500, 32
    sizes = rng.integers(1, 100, n).astype(np.int32)
    lens = np.minimum(sizes, k).astype(np.int32)
    lens[rng.random(n) < 0.1] = 1
    us = rng.integers(0, n, count).astype(np.int32)
    vs = rng.integers(0, n, count).astype(np.int32)
    vs[rng.random(count) < 0.05] = -1
    t = {name: torch.from_numpy(a).cuda() for name, a in (("us", us), ("vs", vs), ("sizes", sizes), ("lens", lens))}
    pu, pv = torch.empty_like(t["us"]), torch.empty_like(t["vs"])
    split = ctypes.c_int64()
    N.call("pg_kmv_merge_partition", N.ptr(t["us"]), N.ptr(t["vs"]), count, N.ptr(t["sizes"]),
           N.ptr(t["lens"]), k, buckets, N.ptr(pu), N.ptr(pv), ctypes.byref(split), N.stream_handle())
    vv = np.maximum(vs, 0)
    keff = np.minimum(lens[us], lens[vv]).astype(np.int64)
    short = (vs >= 0) & ~((sizes[us] <= k) & (sizes[vv] <= k)) & (keff >= 2)
    hu, hv = pu.cpu().numpy(), pv.cpu().numpy()
    s = split.value
    assert s == int(short.sum())
    # stable counting sort: k_eff buckets ascending, then the full merges and pads
    cls = np.where(short, (keff - 1) * buckets // k, buckets)
    order = np.lexsort((np.arange(count), cls))
    assert np.array_equal(hu, us[order]) and np.array_equal(hv, vs[order])


def test_merge_bad_arguments(pg):
    from paper_2208_11469_b200 import _native as N
    from paper_2208_11469_b200.providers import UnsupportedCombinationError
    assert not N.kmv_merge_supported(48) and N.kmv_merge_supported(64)
    with pytest.raises(UnsupportedCombinationError):
        N.call("pg_tc_kmv_merge", None, None, None, 48, None, None, None, 0, 0, None, None)
    with pytest.raises(ValueError):
        N.call("pg_tc_kmv_merge", None, None, None, 64, None, None, None, 3, 1, None, None)
    with pytest.raises(ValueError):
        N.call("pg_tc_kmv_merge", None, None, None, 64, None, None, None, 0, 4, None, None)
