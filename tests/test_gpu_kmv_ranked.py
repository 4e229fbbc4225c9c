"""KMV rank-directory engine (pg_kmv_rank_table, pg_build_kmv_ranked,
pg_tc_kmv_ranked) against the reference semantics.

The engine replaces KMV values by their dense global ranks (a device layout;
the values themselves stay bit-exact) and estimates every edge without
merging the two rows.  Checked here: the rank table against a numpy
restatement of hashing.py:146-153 unit_values; the rank rows against the
values; whole-graph sums against the merge engine and the C oracle's
restatement of providers.py:266-301; and crafted rank rows (dense clusters
that overflow the 3-slot buckets, short rows, verbatim and degenerate
k_eff cases, shared elements) edge by edge against the oracle.
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

RTOL_SUM = 1e-12
INT32_MAX = np.iinfo(np.int32).max
DEFAULT_HASH_SEED = 0x9E3779B97F4A7C15


@pytest.fixture(scope="module")
def pg():
    import paper_2208_11469_b200 as pg
    return pg


def _unit_values(seed0: int, keys: np.ndarray) -> np.ndarray:
    w = O.NumpyPort._hash(seed0, keys)
    out = (w + np.uint64(1)).astype(np.float64)
    out[w == np.uint64(0xFFFFFFFFFFFFFFFF)] = 2.0 ** 64
    return out * 2.0 ** -64


@pytest.mark.parametrize("n", [1, 2, 33, 5000, 70001])
def test_rank_table(pg, n):
    import torch
    from paper_2208_11469_b200 import _native as N
    seeds = O.C.seeds(DEFAULT_HASH_SEED, 1)
    sd = torch.from_numpy(seeds.view(np.int64)).cuda()
    rank_of = torch.empty(n, dtype=torch.int32, device="cuda")
    rank_values = torch.empty(n, dtype=torch.float64, device="cuda")
    N.call("pg_kmv_rank_table", n, N.ptr(sd), N.ptr(rank_of), N.ptr(rank_values),
           N.stream_handle())
    vals = _unit_values(int(seeds[0]), np.arange(n, dtype=np.int64))
    uniq = np.unique(vals)
    want = np.searchsorted(uniq, vals)
    got = rank_of.cpu().numpy()
    assert np.array_equal(got, want)
    rv = rank_values.cpu().numpy()[:len(uniq)]
    assert np.array_equal(rv.view(np.uint64), uniq.view(np.uint64))


@pytest.mark.parametrize("k", [16, 32, 64, 128])
def test_rank_rows_match_values(pg, k):
    g = pg.generate_kronecker(11, 16, 3)
    sk = pg.build_sketched_graph(g, "kmv", s=1.0, k_override=k)
    d = sk.device_tensors()
    ranks = d["ranks"].cpu().numpy()
    rv = d["rank_values"].cpu().numpy()
    vals, lens = sk.values, sk.lengths
    ov, ol = O.C.build_kmv(g.offsets, g.adjacency, k)
    assert np.array_equal(vals, ov) and np.array_equal(lens, ol)
    col = np.arange(k)[None, :]
    inside = col < lens[:, None]
    assert np.all(ranks[~inside] == INT32_MAX)
    assert np.all(np.diff(np.where(inside, ranks, INT32_MAX), axis=1) >= 0)
    got = np.where(inside, rv[np.where(inside, ranks, 0)], np.inf)
    assert np.array_equal(got.view(np.uint64), vals.view(np.uint64))


@pytest.mark.parametrize("graph", ["rmat11", "rmat13", "star", "er"])
@pytest.mark.parametrize("k", [16, 32, 64, 128])
def test_ranked_tc_vs_merge_engine_and_oracle(pg, graph, k):
    import torch
    from paper_2208_11469_b200 import _native as N
    from paper_2208_11469_b200.mining import tc_counts
    if graph == "rmat11":
        g = pg.generate_kronecker(11, 16, 7)
    elif graph == "rmat13":
        g = pg.generate_kronecker(13, 8, 8)
    elif graph == "star":  # one hub over two cliques of small vertices
        e = [[0, i] for i in range(1, 400)]
        e += [[i, j] for i in range(1, 40) for j in range(i + 1, 40)]
        e += [[i, i + 1] for i in range(40, 399)]
        g = pg.CsrGraph.from_edges(e, 400)
    else:
        g = pg.generate_erdos_renyi_gnm(3000, 60000, 4)
    sk = pg.build_sketched_graph(g, "kmv", s=1.0, k_override=k)
    p = pg.make_provider("kmv", sketched=sk)
    got = p._tc_combine(tc_counts(p, g.device()).cpu().numpy())
    # the values merge engine over the same sketches
    us, vs = g.device().upper_edges()
    d = sk.device_tensors()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    N.call("pg_tc_kmv", N.ptr(d["values"]), N.ptr(d["lengths"]), k, N.ptr(d["sizes"]),
           N.ptr(us), N.ptr(vs), 0, us.numel(), N.ptr(out), N.stream_handle())
    merge = float(out.item())
    e = g.edges()
    _, _, est = O.C.pairs_kmv(sk.values, sk.lengths, k, np.diff(g.offsets), e[:, 0], e[:, 1])
    want = float(np.sum(est))
    assert got == pytest.approx(want, rel=RTOL_SUM, abs=1e-9)
    assert merge == pytest.approx(want, rel=RTOL_SUM, abs=1e-9)
    assert pg.tc_estimate(g, sk, "kmv") == pytest.approx(want / 3.0, rel=RTOL_SUM, abs=1e-9)


def _crafted(k, n_rows, rng):
    """Rank rows with the shapes that stress the directory: dense clusters
    (several elements per bucket), a tiny span, short rows, empty rows and
    shared elements between rows."""
    pool_hi = 50_000
    rows = np.full((n_rows, k), INT32_MAX, dtype=np.int64)
    lens = np.zeros(n_rows, dtype=np.int64)
    shared = np.sort(rng.choice(pool_hi, size=3 * k, replace=False))
    for r in range(n_rows):
        kind = r % 6
        if kind == 0:    # spread, overlapping the shared pool
            pick = np.concatenate([rng.choice(shared, k // 2, replace=False),
                                   rng.choice(pool_hi, k, replace=False)])
        elif kind == 1:  # dense cluster: a narrow band holds most elements
            base = int(rng.integers(0, pool_hi - 4 * k))
            pick = np.concatenate([base + rng.choice(2 * k, (3 * k) // 4, replace=False),
                                   rng.choice(pool_hi, k, replace=False)])
        elif kind == 2:  # tiny span: consecutive ranks
            base = int(rng.integers(0, pool_hi - k))
            pick = base + np.arange(k)
        elif kind == 3:  # short row
            pick = rng.choice(shared, int(rng.integers(1, 5)), replace=False)
        elif kind == 4:  # empty row
            pick = np.empty(0, dtype=np.int64)
        else:            # k/2 elements
            pick = rng.choice(pool_hi, k // 2, replace=False)
        pick = np.unique(pick)[:k]
        rows[r, :len(pick)] = pick
        lens[r] = len(pick)
    return rows, lens


@pytest.mark.parametrize("k", [32, 64, 128])
def test_ranked_crafted_rows_edge_by_edge(pg, k):
    import torch
    from paper_2208_11469_b200 import _native as N
    rng = np.random.default_rng(k)
    n_rows = 48
    ranks, lens = _crafted(k, n_rows, rng)
    # strictly increasing values for ranks 0..pool (not uniform: the
    # directory must not rely on the spacing)
    rank_values = np.cumsum(rng.random(60_000) ** 3 + 1e-9) * 1e-5
    vals = np.where(ranks == INT32_MAX, np.inf, rank_values[np.minimum(ranks, 59_999)])
    # sizes: some verbatim (<= k), some not
    sizes = np.where(np.arange(n_rows) % 3 == 0, lens,
                     lens + rng.integers(1, 10 * k, n_rows)).astype(np.int64)
    pairs = np.array([(u, v) for u in range(n_rows) for v in range(n_rows) if u != v])
    pad = N.kmv_ranked_pad(k)
    # one padded group per edge: slots (u, v), (u, -1) x (pad - 1)
    us = np.repeat(pairs[:, 0], pad).astype(np.int32)
    vs = np.full(len(pairs) * pad, -1, dtype=np.int32)
    vs[::pad] = pairs[:, 1]
    dev = {name: torch.from_numpy(np.ascontiguousarray(a)).cuda() for name, a in (
        ("ranks", ranks.astype(np.int32)), ("rv", rank_values), ("lens", lens.astype(np.int32)),
        ("sizes", sizes.astype(np.int32)), ("us", us), ("vs", vs))}
    out = torch.empty(1, dtype=torch.float64, device="cuda")

    def run(b, e):
        N.call("pg_tc_kmv_ranked", N.ptr(dev["ranks"]), N.ptr(dev["rv"]), N.ptr(dev["lens"]), k,
               N.ptr(dev["sizes"]), N.ptr(dev["us"]), N.ptr(dev["vs"]), b, e, N.ptr(out),
               N.stream_handle())
        return float(out.item())

    _, _, est = O.C.pairs_kmv(vals, lens, k, sizes, pairs[:, 0], pairs[:, 1])
    assert run(0, len(us)) == pytest.approx(float(np.sum(est)), rel=RTOL_SUM)
    for i in rng.choice(len(pairs), 120, replace=False):
        assert run(int(i) * pad, int(i + 1) * pad) == est[i], (pairs[i], lens[pairs[i]], sizes[pairs[i]])


def test_ranked_bad_arguments(pg):
    from paper_2208_11469_b200 import _native as N
    from paper_2208_11469_b200.providers import UnsupportedCombinationError
    assert N.kmv_ranked_pad(48) == 0
    with pytest.raises(UnsupportedCombinationError):
        N.call("pg_tc_kmv_ranked", None, None, None, 48, None, None, None, 0, 0, None, None)
    with pytest.raises(ValueError):
        N.call("pg_tc_kmv_ranked", None, None, None, 64, None, None, None, 1, 4, None, None)
