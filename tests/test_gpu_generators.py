"""Device graph generators are bit-identical to the host restatements
(which tests/test_oracle_golden.py and make_golden.py tie to the reference
generate_kronecker)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale,ef,seed", [(1, 4, 0), (8, 16, 3), (14, 16, 2), (16, 8, 7)])
def test_rmat_device_equals_host(scale, ef, seed):
    import paper_2208_11469_b200 as pg
    h = pg.generate_kronecker(scale, ef, seed, device=False)
    d = pg.generate_kronecker(scale, ef, seed, device=True)
    assert np.array_equal(h.offsets, d.offsets)
    assert np.array_equal(h.adjacency, d.adjacency.astype(np.int64))
    # the device mirror is the same graph
    assert np.array_equal(d.device().adj.cpu().numpy(), d.adjacency)


@pytest.mark.parametrize("n,avg,seed", [(4096, 16, 3), (1 << 16, 32, 3)])
def test_chung_lu_device_equals_host(n, avg, seed):
    import paper_2208_11469_b200 as pg
    h = pg.generate_chung_lu(n, avg, 2.1, seed, device=False)
    d = pg.generate_chung_lu(n, avg, 2.1, seed, device=True)
    assert np.array_equal(h.offsets, d.offsets)
    assert np.array_equal(h.adjacency, d.adjacency.astype(np.int64))


def test_pcg64_uniform_matches_numpy():
    import torch
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import _native as N
    from paper_2208_11469_b200.graphs import _pcg64_state
    rng = np.random.default_rng(12345)
    st = _pcg64_state(rng)
    want = rng.random(5000)
    out = torch.empty(3000, dtype=torch.float64, device="cuda")
    N.call("pg_pcg64_uniform", *st, 2000, 3000, N.ptr(out), N.stream_handle())
    assert np.array_equal(out.cpu().numpy(), want[2000:])


@pytest.mark.parametrize("make", [lambda pg: pg.generate_kronecker(16, 16, 9),
                                  lambda pg: pg.generate_erdos_renyi_gnm(3000, 20000, 4),
                                  lambda pg: pg.CsrGraph.from_edges(np.empty((0, 2), np.int64), 17),
                                  lambda pg: pg.CsrGraph.from_edges([[0, 1], [1, 2], [2, 0], [5, 6]], 9)])
def test_degree_order_device_matches_host(make):
    """pg_degree_order == the host restatement of reference graphs.py:154-166
    (rank by (degree, id), N+ keeps higher ranks, adjacency order kept)."""
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200.graphs import _degree_order_host
    g = make(pg)
    want = _degree_order_host(g)
    got = pg.degree_order(g)
    assert got._dev, "device path expected on a CUDA machine"
    for f in ("rank", "offsets", "adjacency"):
        assert np.array_equal(getattr(got, f), getattr(want, f)), f
    assert got.adjacency.dtype == want.adjacency.dtype
    d = got.device()
    assert np.array_equal(d.offsets.cpu().numpy(), want.offsets)
    assert np.array_equal(d.adj.cpu().numpy(), want.adjacency)
    if g.m:
        ex = pg.make_provider("exact_merge", view=got)
        assert pg.triangle_count(got, ex) == pg.triangle_count(want, pg.make_provider("exact_merge", view=want))


@pytest.mark.parametrize("edges,n", [
    ([[0, 1], [1, 0], [2, 2], [3, 1], [1, 3], [1, 3]], None),
    ([[4, 4], [4, 4]], None),
    ([[4, 4], [1, 2]], 9),
    ([[0, 5]], 6),
])
def test_from_edges_device_matches_host(edges, n):
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import graphs
    g = pg.CsrGraph.from_edges(edges, n)
    assert g._dev is not None or g.m == 0
    e = np.asarray(edges, dtype=np.int64)
    # host restatement (the reference's algorithm): canonical unique pairs
    lo, hi = np.minimum(e[:, 0], e[:, 1]), np.maximum(e[:, 0], e[:, 1])
    keep = lo != hi
    uv = np.unique(np.stack([lo[keep], hi[keep]], 1), axis=0)
    nn = n if n is not None else (int(uv.max()) + 1 if len(uv) else 0)
    want = graphs.CsrGraph._from_canonical_keys(uv[:, 0] * nn + uv[:, 1], nn) if len(uv) else None
    assert g.n == nn
    assert g.self_loops_dropped == int((~keep).sum())
    assert g.duplicates_dropped == int(keep.sum()) - len(uv)
    if want is not None:
        assert np.array_equal(g.offsets, want.offsets)
        assert np.array_equal(g.adjacency, want.adjacency)
        assert g.adjacency.dtype == np.int64


def test_from_edges_device_large_and_errors():
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import graphs
    rng = np.random.default_rng(11)
    e = rng.integers(0, 50_000, size=(400_000, 2))
    g = pg.CsrGraph.from_edges(e)
    lo, hi = np.minimum(e[:, 0], e[:, 1]), np.maximum(e[:, 0], e[:, 1])
    keep = lo != hi
    key = np.unique(lo[keep] * g.n + hi[keep])
    want = graphs.CsrGraph._from_canonical_keys(key, g.n)
    assert np.array_equal(g.offsets, want.offsets) and np.array_equal(g.adjacency, want.adjacency)
    assert np.array_equal(g.device().adj.cpu().numpy(), want.adjacency)
    with pytest.raises(ValueError):
        pg.CsrGraph.from_edges([[0, 7]], 5)
    with pytest.raises(ValueError):
        pg.CsrGraph.from_edges([[-1, 2]])
