"""Out-of-bounds write checks through the C ABI (compute-sanitizer is closed
on this GPU pool; profiles/r02_sanitizer.md).

Every output buffer is allocated with a guard region before and after it,
filled with a canary pattern; after the call (and a device sync) both guards
must be intact and the result must equal the unguarded call's.  Inputs are
R-MAT graphs with hub vertices (d > 1024, the builders' hub passes), odd
vertex counts and odd row widths, and edge lists with ragged lengths.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes on each side
CANARY = 0xA5


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import _native as N
    g = pg.generate_kronecker(14, 16, 3)
    dev = g.device()
    assert int(dev.degrees.max()) > 1024
    return pg, N, torch, g, dev


class Guarded:
    """A device buffer of `nbytes` inside canary-filled guard regions."""

    def __init__(self, torch, nbytes):
        self.torch = torch
        self.nbytes = nbytes
        self.buf = torch.full((GUARD + nbytes + GUARD,), CANARY, dtype=torch.uint8, device="cuda")

    @property
    def ptr(self):
        return self.buf.data_ptr() + GUARD

    def check(self):
        self.torch.cuda.synchronize()
        head = self.buf[:GUARD]
        tail = self.buf[GUARD + self.nbytes:]
        assert bool((head == CANARY).all()), "write before the buffer"
        assert bool((tail == CANARY).all()), "write past the buffer"

    def array(self, dtype):
        return self.buf[GUARD:GUARD + self.nbytes].cpu().numpy().view(dtype)


def seeds(torch, count):
    from paper_2208_11469_b200.hashing import HashFamily
    return torch.from_numpy(HashFamily(count=count).seeds_array().view(np.int64)).cuda()


@pytest.mark.parametrize("bits,b", [(576, 3), (1024, 2), (2048, 2), (64, 1)])
def test_build_bloom_guarded(env, bits, b):
    pg, N, torch, g, dev = env
    n = g.n
    words = bits // 64
    rows = Guarded(torch, n * words * 8)
    ones = Guarded(torch, n * 4)
    sd = seeds(torch, b)
    N.call("pg_build_bloom", N.ptr(dev.offsets), N.ptr(dev.adj), n, bits, b, N.ptr(sd),
           rows.ptr, ones.ptr, N.stream_handle())
    rows.check()
    ones.check()
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=b, bits_override=bits)
    assert np.array_equal(rows.array(np.uint64).reshape(n, words), sk.bit_matrix)


@pytest.mark.parametrize("kind,k", [("khash", 32), ("khash", 5), ("onehash", 64), ("onehash", 7),
                                    ("kmv", 64), ("kmv", 3)])
def test_build_minhash_guarded(env, kind, k):
    pg, N, torch, g, dev = env
    n = g.n
    sd = seeds(torch, k if kind == "khash" else 1)
    lengths = Guarded(torch, n * 4)
    if kind == "kmv":
        out = Guarded(torch, n * k * 8)
        N.call("pg_build_kmv", N.ptr(dev.offsets), N.ptr(dev.adj), n, k, N.ptr(sd), out.ptr,
               lengths.ptr, N.stream_handle())
        lengths.check()
    elif kind == "onehash":
        out = Guarded(torch, n * k * 4)
        N.call("pg_build_onehash", N.ptr(dev.offsets), N.ptr(dev.adj), n, k, N.ptr(sd), out.ptr,
               lengths.ptr, N.stream_handle())
        lengths.check()
    else:
        out = Guarded(torch, n * k * 4)
        N.call("pg_build_khash", N.ptr(dev.offsets), N.ptr(dev.adj), n, k, N.ptr(sd), out.ptr,
               N.stream_handle())
    out.check()


@pytest.mark.parametrize("bits", [1024, 2048, 576])
def test_tc_bloom_hist_guarded(env, bits):
    pg, N, torch, g, dev = env
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=bits)
    p = pg.make_provider("bf_and", sketched=sk)
    lay = p._tc_layout(dev)
    hist = Guarded(torch, (bits + 2) * 8)
    d = sk.device_tensors()
    N.call("pg_tc_bloom", N.ptr(d["rows"]), bits, N.PG_BF_AND, N.ptr(d["sizes"]),
           N.ptr(p.lut_device()), N.ptr(lay.us), N.ptr(lay.vs), 0, lay.slots, int(lay.padded),
           hist.ptr, hist.ptr + 8 * (bits + 1), N.stream_handle())
    hist.check()
    assert np.array_equal(hist.array(np.int64)[:bits + 1],
                          p._tc_counts_layout(lay, 0, lay.slots).cpu().numpy()[:bits + 1])


@pytest.mark.parametrize("kind,k", [("bloom", 2048), ("khash", 32), ("onehash", 64), ("kmv", 64)])
def test_pairs_guarded_ragged(env, kind, k):
    pg, N, torch, g, dev = env
    from oracle import oracle as O
    us, vs = O.upper_edges(g.offsets, g.adjacency)
    cnt = 1001  # not a multiple of any lane-group size
    du = torch.from_numpy(us[:cnt].astype(np.int32)).cuda()
    dv = torch.from_numpy(vs[:cnt].astype(np.int32)).cuda()
    est = Guarded(torch, cnt * 8)
    cnts = Guarded(torch, cnt * 4)
    if kind == "bloom":
        sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=k)
        p = pg.make_provider("bf_and", sketched=sk)
        d = sk.device_tensors()
        N.call("pg_pairs_bloom", N.ptr(d["rows"]), k, 2, N.PG_BF_AND, N.ptr(d["sizes"]),
               N.ptr(p.lut_device()), N.ptr(du), N.ptr(dv), cnt, cnts.ptr, est.ptr, N.stream_handle())
    elif kind == "kmv":
        sk = pg.build_sketched_graph(g, "kmv", s=1.0, k_override=k)
        p = pg.make_provider("kmv", sketched=sk)
        d = sk.device_tensors()
        N.call("pg_pairs_kmv", N.ptr(d["values"]), N.ptr(d["lengths"]), k, N.ptr(d["sizes"]),
               N.ptr(du), N.ptr(dv), cnt, cnts.ptr, None, None, est.ptr, N.stream_handle())
    else:
        sk = pg.build_sketched_graph(g, kind, s=1.0, k_override=k)
        p = pg.make_provider(kind, sketched=sk)
        d = sk.device_tensors()
        N.call("pg_pairs_minhash", N.ptr(d["entries"]), k, int(kind == "onehash"),
               N.ptr(d["sizes"]), N.ptr(du), N.ptr(dv), cnt, cnts.ptr, est.ptr, N.stream_handle())
    est.check()
    cnts.check()
    assert np.array_equal(est.array(np.float64), p.pair_many(us[:cnt], vs[:cnt]))


def test_4clique_sketch_workspace_guarded(env):
    """The sketch 4-clique kernel's caller-allocated workspace (partials,
    global C3 scratch) and outputs stay within their sizes, also on the
    global-scratch path."""
    import os
    pg, N, torch, g, dev = env
    view = pg.degree_order(g)
    vdev = view.device()
    for cap in ("512", "4"):
        os.environ["PG_C4S_CAP"] = cap
        try:
            for kind, code in (("khash", N.PG_KHASH), ("onehash", N.PG_ONEHASH), ("kmv", N.PG_KMV)):
                dsk = pg.build_sketched_graph(g, kind, s=1.0, k_override=16, source="directed",
                                              view=view)
                d = dsk.device_tensors()
                maxd = vdev.max_degree()
                wsb = ctypes.c_size_t()
                N.call("pg_4clique_sketch_workspace_size", code, 16, maxd, ctypes.byref(wsb))
                ws = Guarded(torch, wsb.value)
                outs = Guarded(torch, 16)
                rows = d["values"] if kind == "kmv" else d["entries"]
                N.call("pg_4clique_sketch", code, N.ptr(vdev.offsets), N.ptr(vdev.adj),
                       N.ptr(vdev.row_sources()), None, 0, vdev.nnz, N.ptr(rows),
                       N.ptr(d["lengths"]) if kind != "khash" else None, N.ptr(d["sizes"]), 16,
                       N.ptr(d["seeds"]), maxd, ws.ptr, wsb.value, outs.ptr, outs.ptr + 8,
                       N.stream_handle())
                ws.check()
                outs.check()
        finally:
            os.environ.pop("PG_C4S_CAP")
