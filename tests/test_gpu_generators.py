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
