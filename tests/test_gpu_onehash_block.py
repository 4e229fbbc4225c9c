"""1-Hash TC on the per-warp-table engine (onehash_block_kernel: row-padded
slots of pad 256/k, one u table per warp, slot blocks) against the C
oracle's restatement of providers.py:205-232 (_matches_onehash and the
estimate) over the same bit-identical sketches, at every width the engine
takes, on graphs with hubs, short rows, isolated vertices and runs of one
edge; and the exact integer statistics against the unpadded engine."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    import paper_2208_11469_b200 as pg
    return pg


def _graphs(pg):
    e = [[0, i] for i in range(1, 300)] + [[i, i + 1] for i in range(300, 700)]
    e += [[i, j] for i in range(1, 30) for j in range(i + 1, 30)]
    return {"rmat12": pg.generate_kronecker(12, 16, 21),
            "er": pg.generate_erdos_renyi_gnm(4000, 50000, 5),
            "hub_path": pg.CsrGraph.from_edges(e, 800)}


@pytest.mark.parametrize("k", [32, 64, 128])
def test_onehash_block_tc_vs_oracle(pg, k):
    import torch
    from paper_2208_11469_b200 import _native as N
    from paper_2208_11469_b200.mining import tc_counts
    for name, g in _graphs(pg).items():
        sk = pg.build_sketched_graph(g, "onehash", s=1.0, k_override=k)
        ent, ln = O.C.build_onehash(g.offsets, g.adjacency, k)
        assert np.array_equal(sk.entries, ent) and np.array_equal(sk.lengths, ln)
        p = pg.make_provider("onehash", sketched=sk)
        assert p.tc_pad() == N.onehash_block_pad(k)
        counts = tc_counts(p, g.device()).cpu().numpy()
        e = g.edges()
        m = O.C.pairs_minhash(ent, k, True, e[:, 0], e[:, 1])
        sz = np.diff(g.offsets)
        want = float(np.sum(O.minhash_edge_estimates(m, k, sz[e[:, 0]], sz[e[:, 1]], True)))
        assert p._tc_combine(counts) == pytest.approx(want, rel=1e-12, abs=1e-9), name
        # the unpadded engine (plain upper edge list) gives the same integers
        us, vs = g.device().upper_edges()
        d = sk.device_tensors()
        out = torch.empty(2 * k + 3, dtype=torch.int64, device="cuda")
        p0 = N.ptr(out)
        N.call("pg_tc_minhash", N.ptr(d["entries"]), k, 1, N.ptr(d["sizes"]), N.ptr(us), N.ptr(vs), 0,
               us.numel(), 0, p0, p0 + 8 * (k + 1), p0 + 16 * (k + 1), N.stream_handle())
        assert np.array_equal(out.cpu().numpy(), counts), name
