"""Bloom builder at odd row widths (B = 64 x odd, so words64 is odd) and odd
vertex counts, whole-graph and in vertex-range pieces whose row base is only
8-byte aligned -- the layouts where a 16-byte row copy would drop the last
word or fault (reference semantics: sketches.py:314-325, any B that is a
multiple of 64; plan_budget yields such widths)."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    import paper_2208_11469_b200 as pg
    return pg


def _graph(pg, n, seed):
    rng = np.random.default_rng(seed)
    e = rng.integers(0, n, size=(6 * n, 2))
    hub = rng.choice(n, size=min(n - 1, 1500), replace=False)  # one row > 1024 (hub pass)
    e = np.concatenate([e, np.stack([np.zeros(len(hub), np.int64), hub], 1)])
    mid = rng.choice(n, size=min(n - 1, 200), replace=False)  # one 64 < d <= 1024 row
    e = np.concatenate([e, np.stack([np.ones(len(mid), np.int64), mid], 1)])
    e = e[e[:, 0] != e[:, 1]]
    return pg.CsrGraph.from_edges(e, n)


@pytest.mark.parametrize("n", [301, 1999, 2048 + 33])
@pytest.mark.parametrize("bits,b", [(64, 1), (192, 2), (576, 3), (1088, 2), (24640, 2)])
def test_odd_width_whole_graph(pg, n, bits, b):
    g = _graph(pg, n, n + bits)
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=b, bits_override=bits)
    rows, ones = O.C.build_bloom(g.offsets, g.adjacency, bits, b)
    assert np.array_equal(sk.bit_matrix, rows)
    assert np.array_equal(sk.ones, ones)


@pytest.mark.parametrize("bits,b", [(192, 2), (576, 3), (24640, 1)])
def test_odd_width_vertex_range_pieces(pg, bits, b):
    """Build [0, n) as pieces starting at odd vertices through the C ABI: the
    rows pointer of a piece is then 8- but not 16-byte aligned."""
    import torch
    from paper_2208_11469_b200 import _native as N
    n = 1001
    g = _graph(pg, n, 7)
    dev = g.device()
    words = bits // 64
    out = torch.full((n, words), -1, dtype=torch.int64, device="cuda")
    ones = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    seeds = torch.tensor(O.C.seeds(O.DEFAULT_HASH_SEED, b).view(np.int64), device="cuda")
    cuts = [0, 1, 38, 101, 102, 517, n]
    for v0, v1 in zip(cuts[:-1], cuts[1:]):
        N.call("pg_build_bloom", N.ptr(dev.offsets) + 8 * v0, N.ptr(dev.adj), v1 - v0, bits, b,
               N.ptr(seeds), N.ptr(out) + 8 * words * v0, N.ptr(ones) + 4 * v0,
               N.stream_handle())
    torch.cuda.synchronize()
    rows, ones_ref = O.C.build_bloom(g.offsets, g.adjacency, bits, b)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), rows)
    assert np.array_equal(ones.cpu().numpy(), ones_ref)
