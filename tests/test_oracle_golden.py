"""Pin the CPU oracle (oracle/) to outputs of the reference implementation.

The fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  Both restatements -- the C checker and the
numpy port timed as the reference CPU arm -- must reproduce them bit for bit
(integers) and to the last ulp where the reference evaluates the same float
expression.
"""

import numpy as np
import pytest

from conftest import (BLOOM_PARAMS, KS, SMALL_NAMES, SMALL_SEEDS, load_config,
                      sha)
from oracle import oracle as O


def test_hash_kat(hash_kat):
    a = hash_kat["ref_test_anchors"]
    s = O.C.seeds(O.DEFAULT_HASH_SEED, 4)
    assert int(s[0]) == a["seed0"] and int(s[1]) == a["seed1"]
    assert [int(x) for x in s] == hash_kat["seeds_default4"]
    assert [int(x) for x in O.C.seeds(7, 2)] == hash_kat["seeds_seed7"]
    keys = np.asarray(hash_kat["keys"], dtype=np.int64)
    w0 = O.NumpyPort._hash(int(s[0]), keys)
    w3 = O.NumpyPort._hash(int(s[3]), keys)
    assert [int(x) for x in w0] == hash_kat["words_default_fn0"]
    assert [int(x) for x in w3] == hash_kat["words_default_fn3"]
    assert int(O.NumpyPort._hash(int(s[0]), np.asarray([12345]))[0]) % 256 == a["bit_0_12345_256"]
    assert int(O.NumpyPort._hash(int(s[1]), np.asarray([12345]))[0]) % 256 == a["bit_1_12345_256"]
    s7 = O.C.seeds(7, 2)
    assert int(O.NumpyPort._hash(int(s7[0]), np.asarray([0]))[0]) % 65536 == a["fam7_bit_0_0_65536"]


def _graph(golden, name):
    return golden[f"{name}/offsets"], golden[f"{name}/adjacency"]


@pytest.mark.parametrize("name", SMALL_NAMES)
@pytest.mark.parametrize("bits,b", BLOOM_PARAMS)
def test_c_oracle_bloom_small(small_golden, name, bits, b):
    off, adj = _graph(small_golden, name)
    key = f"{name}/bloom{bits}_{b}"
    rows, ones = O.C.build_bloom(off, adj, bits, b, SMALL_SEEDS[name] + 100)
    assert np.array_equal(rows, small_golden[f"{key}/bit_matrix"])
    assert np.array_equal(ones, small_golden[f"{key}/ones"])
    us, vs = O.upper_edges(off, adj)
    sizes = np.diff(off)
    for kind in ("bf_and", "bf_l", "bf_or"):
        pop = O.C.pairs_bloom(rows, bits, kind == "bf_or", us, vs)
        est = O.bloom_edge_estimates(pop, kind, bits, b, sizes[us], sizes[vs])
        assert np.array_equal(est, small_golden[f"{key}/pairs_{kind}"]), kind
        tc = O.NumpyPort(threads=1).tc_sum(
            lambda a, c: O.NumpyPort.bloom_chunk(rows, bits, b, kind, sizes, a, c), us, vs) / 3.0
        assert tc == pytest.approx(small_golden[f"{key}/tc_{kind}"][0], rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("name", SMALL_NAMES)
@pytest.mark.parametrize("bits,b", BLOOM_PARAMS)
def test_numpy_port_bloom_build(small_golden, name, bits, b):
    off, adj = _graph(small_golden, name)
    rows, ones = O.NumpyPort().build_bloom(off, adj, bits, b, SMALL_SEEDS[name] + 100)
    key = f"{name}/bloom{bits}_{b}"
    assert np.array_equal(rows, small_golden[f"{key}/bit_matrix"])
    assert np.array_equal(ones, small_golden[f"{key}/ones"])


@pytest.mark.parametrize("name", SMALL_NAMES)
@pytest.mark.parametrize("k", KS)
def test_c_oracle_minhash_kmv_small(small_golden, name, k):
    off, adj = _graph(small_golden, name)
    seed = SMALL_SEEDS[name] + 300
    us, vs = O.upper_edges(off, adj)
    sizes = np.diff(off)
    ent = O.C.build_khash(off, adj, k, seed)
    assert np.array_equal(ent, small_golden[f"{name}/khash{k}/entries"])
    m = O.C.pairs_minhash(ent, k, False, us, vs)
    est = O.minhash_edge_estimates(m, k, sizes[us], sizes[vs], False)
    assert np.array_equal(est, small_golden[f"{name}/khash{k}/pairs"])
    assert np.array_equal(O.NumpyPort.khash_chunk(ent, k, sizes, us, vs), est)

    ent1, ln1 = O.C.build_onehash(off, adj, k, seed)
    assert np.array_equal(ent1, small_golden[f"{name}/onehash{k}/entries"])
    assert np.array_equal(ln1, small_golden[f"{name}/onehash{k}/lengths"])
    m1 = O.C.pairs_minhash(ent1, k, True, us, vs)
    est1 = O.minhash_edge_estimates(m1, k, sizes[us], sizes[vs], True)
    assert np.array_equal(est1, small_golden[f"{name}/onehash{k}/pairs"])
    assert np.array_equal(O.NumpyPort.onehash_chunk(ent1, k, sizes, us, vs), est1)

    val, lnv = O.C.build_kmv(off, adj, k, seed)
    assert np.array_equal(val, small_golden[f"{name}/kmv{k}/values"])
    assert np.array_equal(lnv, small_golden[f"{name}/kmv{k}/lengths"])
    _, _, estv = O.C.pairs_kmv(val, lnv, k, sizes, us, vs)
    assert np.array_equal(estv, small_golden[f"{name}/kmv{k}/pairs"])
    assert np.array_equal(O.NumpyPort.kmv_chunk(val, lnv, k, sizes, us, vs), estv)


@pytest.mark.parametrize("name", SMALL_NAMES)
def test_c_oracle_exact_and_4clique(small_golden, name):
    off, adj = _graph(small_golden, name)
    us, vs = O.upper_edges(off, adj)
    ex = O.C.pairs_exact(off, adj, us, vs)
    assert np.array_equal(ex, small_golden[f"{name}/pairs_exact"])
    assert ex.sum() == 3 * small_golden[f"{name}/tc_exact"][0]


def _er_c1():
    from paper_2208_11469_b200.graphs import generate_erdos_renyi_gnm
    return generate_erdos_renyi_gnm(16384, 262144, 0)


def test_config1_graph_and_bloom():
    cfg = load_config("config1.json")
    g = _er_c1()
    assert g.m == cfg["m"] == 262144
    assert sha(g.offsets.astype("<i8")) == cfg["offsets_sha"]
    assert sha(g.adjacency.astype("<i8")) == cfg["adjacency_sha"]
    rec = cfg["sketches"]["bloom512_1"]
    rows, ones = O.C.build_bloom(g.offsets, g.adjacency, 512, 1)
    assert sha(rows.astype("<u8")) == rec["bit_matrix"]
    assert sha(ones.astype("<i8")) == rec["ones"]
    us, vs = O.upper_edges(g.offsets, g.adjacency)
    pop = O.C.pairs_bloom(rows, 512, False, us, vs)
    assert np.bincount(pop, minlength=513).tolist() == rec["and_popcount_hist"]
    sizes = np.diff(g.offsets)
    for kind, want in rec["tc"].items():
        got = O.NumpyPort(threads=4).tc_sum(
            lambda a, c: O.NumpyPort.bloom_chunk(rows, 512, 1, kind, sizes, a, c), us, vs) / 3.0
        assert got == pytest.approx(want, rel=1e-12)


def test_config1_minhash_kmv():
    cfg = load_config("config1.json")
    g = _er_c1()
    sk = cfg["sketches"]
    ent = O.C.build_khash(g.offsets, g.adjacency, 32)
    assert sha(ent.astype("<i8")) == sk["khash32"]["entries"]
    us, vs = O.upper_edges(g.offsets, g.adjacency)
    m = O.C.pairs_minhash(ent, 32, False, us, vs)
    assert np.bincount(m, minlength=33).tolist() == sk["khash32"]["match_hist"]
    assert int(np.count_nonzero(m / 32 >= 0.1)) == sk["khash32"]["jaccard_hat_kept"]
    e1, l1 = O.C.build_onehash(g.offsets, g.adjacency, 64)
    assert sha(e1.astype("<i8")) == sk["onehash64"]["entries"]
    assert sha(l1.astype("<i8")) == sk["onehash64"]["lengths"]
    v, lv = O.C.build_kmv(g.offsets, g.adjacency, 64)
    assert sha(v.astype("<f8")) == sk["kmv64"]["values"]
    assert sha(lv.astype("<i8")) == sk["kmv64"]["lengths"]
    sizes = np.diff(g.offsets)
    _, _, est = O.C.pairs_kmv(v, lv, 64, sizes, us, vs)
    assert est.sum() / 3.0 == pytest.approx(sk["kmv64"]["tc"]["kmv"], rel=1e-12)


@pytest.mark.slow
def test_config2_bloom_checksums():
    cfg = load_config("config2.json")
    from paper_2208_11469_b200.graphs import generate_kronecker
    g = generate_kronecker(20, 16, 1)
    assert g.m == cfg["m"]
    assert sha(g.offsets.astype("<i8")) == cfg["offsets_sha"]
    assert sha(g.adjacency.astype("<i8")) == cfg["adjacency_sha"]
    rec = cfg["sketches"]["bloom1024_2"]
    rows, ones = O.C.build_bloom(g.offsets, g.adjacency, 1024, 2)
    assert sha(rows.astype("<u8")) == rec["bit_matrix"]
    assert sha(ones.astype("<i8")) == rec["ones"]
    us, vs = O.upper_edges(g.offsets, g.adjacency)
    pop = O.C.pairs_bloom(rows, 1024, False, us, vs)
    hist = np.bincount(pop, minlength=1025)
    assert hist.tolist() == rec["and_popcount_hist"]
    lut = O.swamidass(1024, 2, np.arange(1025))
    import math
    got = math.fsum(float(h) * float(l) for h, l in zip(hist, lut) if h) / 3.0
    assert got == pytest.approx(rec["tc"]["bf_and"], rel=1e-12)


def test_oracle_rmat_generator_s20():
    """The oracle's C restatement of generate_kronecker (graphs.py:251-276,
    PCG64 draws + CsrGraph.from_edges) reproduces the reference's s20 seed 1
    CSR byte for byte (config2.json, written by the reference)."""
    import hashlib
    from conftest import load_config
    from oracle import oracle as O
    cfg = load_config("config2.json")
    off, adj = O.C.generate_kronecker(20, 16, 1)
    assert len(adj) // 2 == cfg["m"]
    assert hashlib.sha256(off.astype("<i8").tobytes()).hexdigest() == cfg["offsets_sha"]
    assert hashlib.sha256(adj.astype("<i8").tobytes()).hexdigest() == cfg["adjacency_sha"]


def test_oracle_rmat_generator_small_matches_numpy():
    """Small scales against the numpy restatement of the same draws."""
    from oracle import oracle as O
    from paper_2208_11469_b200 import graphs as G
    for scale, ef, seed in ((1, 2, 0), (5, 3, 7), (10, 16, 3)):
        off, adj = O.C.generate_kronecker(scale, ef, seed)
        g = G.generate_kronecker(scale, ef, seed, device=False)
        assert np.array_equal(off, g.offsets) and np.array_equal(adj, g.adjacency)
