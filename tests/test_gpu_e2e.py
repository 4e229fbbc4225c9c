"""The end-to-end host-input path: chunked pinned upload overlapped with the
sketch build (graphs.DeviceCsr._chunked_upload, sketches._build_on_device)
must give bit-identical sketches and estimates to the plain path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pinned(a):
    import torch
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def _device_arrays(sk):
    return {k: v.cpu().numpy() for k, v in sk.device_tensors().items()}


@pytest.mark.parametrize("kind,kw", [("bloom", {"bits_override": 1024, "b": 2}),
                                     ("bloom", {"bits_override": 2048, "b": 1}),
                                     ("khash", {"k_override": 32}),
                                     ("onehash", {"k_override": 64}),
                                     ("kmv", {"k_override": 64})])
@pytest.mark.parametrize("chunks", [1, 3, 8, 64])
def test_chunked_upload_build_identical(monkeypatch, kind, kw, chunks):
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import graphs
    g = pg.generate_kronecker(14, 16, 7)  # R-MAT hubs + isolated vertices
    ref = pg.build_sketched_graph(g, kind, s=1.0, **kw)
    want = _device_arrays(ref)
    monkeypatch.setattr(graphs, "CHUNKED_UPLOAD_MIN_BYTES", 0)
    monkeypatch.setattr(graphs, "UPLOAD_CHUNKS", chunks)
    hg = pg.CsrGraph(_pinned(g.offsets), _pinned(g.adjacency.astype(np.int32)))
    dev = hg.device()
    assert dev.upload_chunks, "pinned int32 input must take the chunked path"
    got_sk = pg.build_sketched_graph(hg, kind, s=1.0, **kw)
    assert not dev.upload_chunks
    got = _device_arrays(got_sk)
    assert sorted(got) == sorted(want)
    for key in want:
        assert np.array_equal(got[key], want[key]), key
    est_kind = {"bloom": "bf_and"}.get(kind, kind)
    # integer reductions are exact; KMV's fp64 sum is order-dependent in the last bits
    assert pg.tc_estimate(hg, got_sk, est_kind) == pytest.approx(
        pg.tc_estimate(g, ref, est_kind), rel=1e-12)
    # a second sketch of the same (already resident) graph uses the plain path
    again = pg.build_sketched_graph(hg, kind, s=1.0, **kw)
    for key, v in _device_arrays(again).items():
        assert np.array_equal(v, want[key]), key


def test_chunked_upload_csr_identical(monkeypatch):
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import graphs
    g = pg.generate_erdos_renyi_gnm(5000, 40000, 3)
    monkeypatch.setattr(graphs, "CHUNKED_UPLOAD_MIN_BYTES", 0)
    hg = pg.CsrGraph(_pinned(g.offsets), _pinned(g.adjacency.astype(np.int32)))
    dev = hg.device()
    assert np.array_equal(dev.offsets.cpu().numpy(), g.offsets)
    assert np.array_equal(dev.adj.cpu().numpy(), g.adjacency)
    us, vs = dev.upper_edges()
    e = g.edges()
    assert np.array_equal(us.cpu().numpy(), e[:, 0]) and np.array_equal(vs.cpu().numpy(), e[:, 1])


def test_bloom_hub_slices_match_oracle():
    """Rows of hub vertices (degree > 1024, built in 2048-entry slices by many
    CTAs with global atomics) equal the oracle's rows."""
    import paper_2208_11469_b200 as pg
    from oracle import oracle as O
    n = 9000
    # vertex 0 adjacent to everything, vertex 1 to the even vertices, a ring
    src = [np.zeros(n - 1, np.int64), np.ones(len(range(2, n, 2)), np.int64),
           np.arange(2, n - 1, dtype=np.int64)]
    dst = [np.arange(1, n, dtype=np.int64), np.arange(2, n, 2, dtype=np.int64),
           np.arange(3, n, dtype=np.int64)]
    g = pg.CsrGraph.from_edges(np.stack([np.concatenate(src), np.concatenate(dst)], 1), n)
    assert g.degree(0) > 4 * 2048
    for bits, b in ((1024, 2), (512, 3), (2048, 1)):
        sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=b, bits_override=bits, seed=11)
        rows, ones = O.C.build_bloom(g.offsets, g.adjacency, bits, b, seed=11)
        assert np.array_equal(sk.bit_matrix, rows)
        assert np.array_equal(sk.ones, ones)


def test_device_seeds_match_host_family():
    import torch
    from paper_2208_11469_b200 import _native as N
    from paper_2208_11469_b200.hashing import HashFamily
    for base, count in ((0x9E3779B97F4A7C15, 1), (17, 64), (2 ** 64 - 1, 33)):
        fam = HashFamily(base_seed=base, count=count)
        out = torch.empty(count, dtype=torch.int64, device="cuda")
        N.call("pg_family_seeds_device", fam.base_seed, count, N.ptr(out), N.stream_handle())
        assert np.array_equal(out.cpu().numpy().view(np.uint64), fam.seeds_array())


@pytest.mark.parametrize("kind,sk_kind,kw", [("bf_and", "bloom", {"bits_override": 512, "b": 2}),
                                             ("khash", "khash", {"k_override": 32}),
                                             ("onehash", "onehash", {"k_override": 32}),
                                             ("kmv", "kmv", {"k_override": 32})])
def test_pair_many_reentrant_from_threads(kind, sk_kind, kw):
    """providers are shared by thread-pool workers that call
    pair_many on disjoint slices concurrently (reference mining.py:75-76)."""
    from concurrent.futures import ThreadPoolExecutor
    import paper_2208_11469_b200 as pg
    g = pg.generate_kronecker(14, 16, 3)
    sk = pg.build_sketched_graph(g, sk_kind, s=1.0, **kw)
    p = pg.make_provider(kind, sketched=sk)
    e = g.edges()
    want = p.pair_many(e[:, 0], e[:, 1])
    cuts = np.linspace(0, len(e), 33).astype(int)

    def work(i):
        return p.pair_many(e[cuts[i]:cuts[i + 1], 0], e[cuts[i]:cuts[i + 1], 1])

    with ThreadPoolExecutor(max_workers=8) as pool:
        parts = list(pool.map(work, range(32)))
    assert np.array_equal(np.concatenate(parts), want)


def test_pair_many_index_rules_match_numpy():
    """Row gathers follow numpy's indexing as in the reference: negative IDs
    wrap, IDs outside [-n, n) raise IndexError (never reach a kernel)."""
    import paper_2208_11469_b200 as pg
    g = pg.CsrGraph.from_edges([[0, 1], [1, 2], [2, 3]])
    for kind, sk_kind in (("bf_and", "bloom"), ("khash", "khash"), ("kmv", "kmv")):
        sk = pg.build_sketched_graph(g, sk_kind, s=1.0, b=1, bits_override=64, k_override=4)
        p = pg.make_provider(kind, sketched=sk)
        assert np.array_equal(p.pair_many(np.array([0, 1]), np.array([-1, -3])),
                              p.pair_many(np.array([0, 1]), np.array([3, 1])))
        for bad in ([4], [-5], [100]):
            with pytest.raises(IndexError):
                p.pair_many(np.array([0]), np.array(bad))
    ex = pg.make_provider("exact_merge", graph=g)
    with pytest.raises(IndexError):
        ex.pair_many(np.array([0]), np.array([4]))
    assert ex.pair_many(np.array([0]), np.array([-2])).tolist() == \
        ex.pair_many(np.array([0]), np.array([2])).tolist()


@pytest.mark.parametrize("pad", [1, 2, 4, 8])
@pytest.mark.parametrize("lower", [0, 1])
def test_range_slots_append_matches_whole_layout(pad, lower):
    """pg_csr_range_slots_append over consecutive vertex ranges (device
    cursor, no host sync) reproduces the whole-graph padded layout range by
    range; lower = 1 gives the mirrored (v < u) slots."""
    import ctypes
    import torch
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import _native as N
    g = pg.generate_kronecker(13, 16, 11)
    dev = g.device()
    off, adj = g.offsets, g.adjacency
    # expected: rows in order, each row's upper (or lower) entries padded to pad
    want_v, want_u = [], []
    for u in range(g.n):
        row = adj[off[u]:off[u + 1]]
        part = row[row < u] if lower else row[row > u]
        c = -(-len(part) // pad) * pad
        want_v += list(part) + [-1] * (c - len(part))
        want_u += [u] * (c // pad)
    cuts = [0, 3, 100, 2000, 2001, 5000, g.n]
    cap = g.offsets[-1] + (pad - 1) * g.n + pad
    ug = torch.full((cap // pad + 1,), -7, dtype=torch.int32, device="cuda")
    vs = torch.full((cap,), -7, dtype=torch.int32, device="cuda")
    cursor = torch.zeros(2 + 2 * len(cuts), dtype=torch.int64, device="cuda")
    for i, (v0, v1) in enumerate(zip(cuts[:-1], cuts[1:])):
        bound = int(off[v1] - off[v0]) + (pad - 1) * (v1 - v0)
        ws_bytes = ctypes.c_size_t()
        N.call("pg_csr_range_slots_workspace", v1 - v0, bound, ctypes.byref(ws_bytes))
        ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device="cuda")
        N.call("pg_csr_range_slots_append", N.ptr(dev.offsets), N.ptr(dev.adj), v0, v1, pad, lower,
               bound, N.ptr(ug), N.ptr(vs), cap, N.ptr(cursor), N.ptr(cursor) + 8 * (2 + 2 * i),
               N.ptr(ws), ws_bytes.value, N.stream_handle())
    c = cursor.cpu().numpy()
    total = len(want_v)
    assert c[0] == total and c[1] == 0
    rng = c[2:2 + 2 * (len(cuts) - 1)].reshape(-1, 2)
    assert rng[0, 0] == 0 and rng[-1, 1] == total and np.all(rng[1:, 0] == rng[:-1, 1])
    assert np.array_equal(vs[:total].cpu().numpy(), np.array(want_v, dtype=np.int32))
    assert np.array_equal(ug[:total // pad].cpu().numpy(), np.array(want_u, dtype=np.int32))


def test_tc_bloom_range_accumulates_to_whole():
    """pg_tc_bloom_range over appended ranges, accumulating, gives the
    whole-graph pg_tc_bloom histogram (same integers)."""
    import ctypes
    import torch
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import _native as N
    g = pg.generate_kronecker(13, 16, 12)
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=1024)
    p = pg.make_provider("bf_and", sketched=sk)
    from paper_2208_11469_b200.mining import tc_counts
    want = tc_counts(p, g.device()).cpu().numpy()
    dev, d = g.device(), sk.device_tensors()
    pad = p.tc_pad()
    cuts = [0, 17, 900, 4000, g.n]
    cap = g.offsets[-1] + (pad - 1) * g.n + pad
    ug = torch.empty(cap // pad + 1, dtype=torch.int32, device="cuda")
    vs = torch.empty(cap, dtype=torch.int32, device="cuda")
    cursor = torch.zeros(2 + 2 * len(cuts), dtype=torch.int64, device="cuda")
    out = torch.zeros(1024 + 2, dtype=torch.int64, device="cuda")
    for i, (v0, v1) in enumerate(zip(cuts[:-1], cuts[1:])):
        bound = int(g.offsets[v1] - g.offsets[v0]) + (pad - 1) * (v1 - v0)
        ws_bytes = ctypes.c_size_t()
        N.call("pg_csr_range_slots_workspace", v1 - v0, bound, ctypes.byref(ws_bytes))
        ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device="cuda")
        rng = N.ptr(cursor) + 8 * (2 + 2 * i)
        N.call("pg_csr_range_slots_append", N.ptr(dev.offsets), N.ptr(dev.adj), v0, v1, pad, 0,
               bound, N.ptr(ug), N.ptr(vs), cap, N.ptr(cursor), rng, N.ptr(ws), ws_bytes.value,
               N.stream_handle())
        N.call("pg_tc_bloom_range", N.ptr(d["rows"]), 1024, p.op, None, None, N.ptr(ug), N.ptr(vs),
               rng, bound, 1, N.ptr(out), N.ptr(out) + 8 * 1025, N.stream_handle())
    assert np.array_equal(out.cpu().numpy(), want)


def test_scalar_sketch_row_does_not_materialise_matrix():
    """sketch(v) (and the scalar with_set / est_* built on it) copies one
    row from the device; the whole host mirror appears only when the
    matrix attribute itself is read (reference sketches.py:282-295)."""
    import paper_2208_11469_b200 as pg
    g = pg.generate_kronecker(12, 16, 1)
    for kind, kw in (("bloom", {"b": 2, "bits_override": 1024}), ("khash", {"k_override": 32}),
                     ("onehash", {"k_override": 32}), ("kmv", {"k_override": 32})):
        sk = pg.build_sketched_graph(g, kind, s=1.0, **kw)
        rows = [sk.sketch(v) for v in (0, 5, g.n - 1, -1)]
        name = {"bloom": "bit_matrix", "khash": "entries", "onehash": "entries",
                "kmv": "values"}[kind]
        assert sk._host.get(name) is None, kind
        full = getattr(sk, name)  # now materialise and compare
        for v, r in zip((0, 5, g.n - 1, -1), rows):
            got = {"bloom": lambda s: s.words, "khash": lambda s: s.entries,
                   "onehash": lambda s: s.entries, "kmv": lambda s: s.hashes}[kind](r)
            want = full[v]
            if kind in ("onehash", "kmv"):
                want = want[:sk.lengths[v]]
            if kind == "khash" and sk.sizes[v] == 0:
                want = want[:0]
            assert np.array_equal(got, want), (kind, v)
