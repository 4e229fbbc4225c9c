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
