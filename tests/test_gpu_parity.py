"""Parity of the CUDA path (through the C ABI) with the reference.

Integer outputs (sketch bits/entries/values, per-edge popcounts and match
counts, histograms) must be bit-exact; per-edge float estimates are required
to be identical (same IEEE expression, no FMA contraction); whole-graph sums
agree within 1e-12 relative (north-star tolerance 1e-6).
"""

import numpy as np
import pytest

from conftest import (BLOOM_PARAMS, KS, SMALL_NAMES, SMALL_SEEDS, load_config,
                      sha, small_graph)
from oracle import oracle as O

pytestmark = pytest.mark.gpu

RTOL_SUM = 1e-12


@pytest.fixture(scope="module")
def pg():
    import paper_2208_11469_b200 as pg
    return pg


@pytest.mark.parametrize("name", SMALL_NAMES)
@pytest.mark.parametrize("bits,b", BLOOM_PARAMS)
def test_bloom_build_pairs_tc(pg, small_golden, name, bits, b):
    gd = small_golden
    g = small_graph(gd, name)
    key = f"{name}/bloom{bits}_{b}"
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=b, seed=SMALL_SEEDS[name] + 100,
                                 bits_override=bits)
    assert np.array_equal(sk.bit_matrix, gd[f"{key}/bit_matrix"])
    assert np.array_equal(sk.ones, gd[f"{key}/ones"])
    e = g.edges()
    for kind in ("bf_and", "bf_l", "bf_or"):
        p = pg.make_provider(kind, sketched=sk)
        est = p.pair_many(e[:, 0], e[:, 1])
        assert np.array_equal(est, gd[f"{key}/pairs_{kind}"]), kind
        tc = pg.tc_estimate(g, sk, kind)
        assert tc == pytest.approx(gd[f"{key}/tc_{kind}"][0], rel=RTOL_SUM, abs=1e-9)
        jp = pg.jarvis_patrick_cluster(g, p, 1.0)
        assert [len(jp.kept_edges), jp.cluster_count, jp.singleton_count] == \
            gd[f"{key}/jp_{kind}"].tolist()
        pop = p.pair_counts(e[:, 0], e[:, 1])
        want = O.C.pairs_bloom(gd[f"{key}/bit_matrix"], bits, kind == "bf_or",
                               e[:, 0], e[:, 1])
        assert np.array_equal(pop, want)


@pytest.mark.parametrize("name", SMALL_NAMES)
@pytest.mark.parametrize("bits,b", BLOOM_PARAMS)
def test_bloom_directed_4clique(pg, small_golden, name, bits, b):
    gd = small_golden
    g = small_graph(gd, name)
    view = pg.degree_order(g)
    key = f"{name}/bloom{bits}_{b}"
    dsk = pg.build_sketched_graph(g, "bloom", s=1.0, b=b, seed=SMALL_SEEDS[name] + 200,
                                  bits_override=bits, source="directed", view=view)
    assert np.array_equal(dsk.bit_matrix, gd[f"{key}/dir_bit_matrix"])
    assert np.array_equal(dsk.sizes, view.out_degrees())
    for kind in ("bf_and", "bf_l"):
        p = pg.make_provider(kind, sketched=dsk)
        got = pg.four_clique_count(view, p)
        assert got == pytest.approx(gd[f"{key}/c4_{kind}"][0], rel=RTOL_SUM, abs=1e-9)


@pytest.mark.parametrize("name", SMALL_NAMES)
def test_exact_paths(pg, small_golden, name):
    gd = small_golden
    g = small_graph(gd, name)
    view = pg.degree_order(g)
    ex = pg.make_provider("exact_merge", view=view)
    assert pg.triangle_count(view, ex) == gd[f"{name}/tc_exact"][0]
    assert pg.four_clique_count(view, ex) == gd[f"{name}/c4_exact"][0]
    e = g.edges()
    exg = pg.make_provider("exact_merge", graph=g)
    assert np.array_equal(exg.pair_many(e[:, 0], e[:, 1]), gd[f"{name}/pairs_exact"])
    assert pg.tc_estimate(g, kind="exact_merge") == float(gd[f"{name}/tc_exact"][0])


@pytest.mark.parametrize("name", SMALL_NAMES)
@pytest.mark.parametrize("k", KS)
@pytest.mark.parametrize("kind", ["khash", "onehash", "kmv"])
def test_minhash_kmv(pg, small_golden, name, k, kind):
    gd = small_golden
    g = small_graph(gd, name)
    key = f"{name}/{kind}{k}"
    sk = pg.build_sketched_graph(g, kind, s=1.0, seed=SMALL_SEEDS[name] + 300, k_override=k)
    if kind == "kmv":
        assert np.array_equal(sk.values, gd[f"{key}/values"])
        assert np.array_equal(sk.lengths, gd[f"{key}/lengths"])
    else:
        assert np.array_equal(sk.entries, gd[f"{key}/entries"])
        if kind == "onehash":
            assert np.array_equal(sk.lengths, gd[f"{key}/lengths"])
    e = g.edges()
    p = pg.make_provider(kind, sketched=sk)
    est = p.pair_many(e[:, 0], e[:, 1])
    assert np.array_equal(est, gd[f"{key}/pairs"])
    assert pg.tc_estimate(g, sk, kind) == pytest.approx(gd[f"{key}/tc"][0], rel=RTOL_SUM, abs=1e-9)
    jp = pg.jarvis_patrick_cluster(g, p, 1.0)
    assert [len(jp.kept_edges), jp.cluster_count, jp.singleton_count] == gd[f"{key}/jp"].tolist()
    if kind == "khash":
        jc = pg.jaccard_cluster_count(g, sk, 0.1)
        assert jc.kept_hat == int(np.count_nonzero(gd[f"{key}/jaccard_hat"] >= 0.1))
        assert jc.kept_similarity == int(np.count_nonzero(gd[f"{key}/jaccard_sim"] >= 0.1))
        assert int(jc.match_hist.sum()) == len(e)


def test_scalar_estimators_match_batch(pg, small_golden):
    gd = small_golden
    g = small_graph(gd, "g60")
    e = g.edges()[:40]
    for kind, sk_kind in (("bf_and", "bloom"), ("bf_l", "bloom"), ("bf_or", "bloom"),
                          ("khash", "khash"), ("onehash", "onehash"), ("kmv", "kmv")):
        sk = pg.build_sketched_graph(g, sk_kind, s=0.9, b=2, seed=17)
        p = pg.make_provider(kind, sketched=sk)
        batch = p.pair_many(e[:, 0], e[:, 1])
        for i, (u, v) in enumerate(e.tolist()):
            assert batch[i] == pytest.approx(p.pair(u, v), rel=1e-12)


def test_config1_full_parity(pg):
    cfg = load_config("config1.json")
    g = pg.generate_erdos_renyi_gnm(16384, 262144, 0)
    assert sha(g.adjacency.astype("<i8")) == cfg["adjacency_sha"]
    rec = cfg["sketches"]["bloom512_1"]
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=1, bits_override=512)
    assert sha(sk.bit_matrix.astype("<u8")) == rec["bit_matrix"]
    assert sha(sk.ones.astype("<i8")) == rec["ones"]
    e = g.edges()
    p = pg.make_provider("bf_and", sketched=sk)
    pop = p.pair_counts(e[:, 0], e[:, 1])
    assert np.bincount(pop, minlength=513).tolist() == rec["and_popcount_hist"]
    for kind, want in rec["tc"].items():
        assert pg.tc_estimate(g, sk, kind) == pytest.approx(want, rel=RTOL_SUM)
    sk = cfg["sketches"]
    kh = pg.build_sketched_graph(g, "khash", s=1.0, k_override=32)
    assert sha(kh.entries.astype("<i8")) == sk["khash32"]["entries"]
    jc = pg.jaccard_cluster_count(g, kh, 0.1)
    assert jc.match_hist.tolist() == sk["khash32"]["match_hist"]
    assert jc.kept_hat == sk["khash32"]["jaccard_hat_kept"]
    assert pg.tc_estimate(g, kh, "khash") == pytest.approx(sk["khash32"]["tc"]["khash"], rel=RTOL_SUM)
    oh = pg.build_sketched_graph(g, "onehash", s=1.0, k_override=64)
    assert sha(oh.entries.astype("<i8")) == sk["onehash64"]["entries"]
    assert sha(oh.lengths.astype("<i8")) == sk["onehash64"]["lengths"]
    assert pg.tc_estimate(g, oh, "onehash") == pytest.approx(sk["onehash64"]["tc"]["onehash"], rel=RTOL_SUM)
    kv = pg.build_sketched_graph(g, "kmv", s=1.0, k_override=64)
    assert sha(kv.values.astype("<f8")) == sk["kmv64"]["values"]
    assert sha(kv.lengths.astype("<i8")) == sk["kmv64"]["lengths"]
    assert pg.tc_estimate(g, kv, "kmv") == pytest.approx(sk["kmv64"]["tc"]["kmv"], rel=RTOL_SUM)


def test_config2_full_parity(pg):
    cfg = load_config("config2.json")
    g = pg.generate_kronecker(20, 16, 1)
    assert sha(g.adjacency.astype("<i8")) == cfg["adjacency_sha"]
    rec = cfg["sketches"]["bloom1024_2"]
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=1024)
    assert sha(sk.bit_matrix.astype("<u8")) == rec["bit_matrix"]
    assert sha(sk.ones.astype("<i8")) == rec["ones"]
    p = pg.make_provider("bf_and", sketched=sk)
    from paper_2208_11469_b200.mining import tc_counts
    counts = tc_counts(p, g.device()).cpu().numpy()
    assert counts[:-1].tolist() == rec["and_popcount_hist"]
    # the general (unpadded) layout and any shard split give the same integers
    us, vs = g.device().upper_edges()
    assert p._tc_counts(us, vs, 0, us.numel()).cpu().numpy().tolist() == counts.tolist()
    parts = sum(tc_counts(p, g.device(), r, 3).cpu().numpy() for r in range(3))
    assert parts.tolist() == counts.tolist()
    for kind, want in rec["tc"].items():
        assert pg.tc_estimate(g, sk, kind) == pytest.approx(want, rel=RTOL_SUM)


@pytest.mark.parametrize("k", [16, 32, 64, 128])
def test_kmv_pairs_all_widths_vs_oracle(pg, k):
    """KMV per-edge estimates for every dispatch width (k = 32/64/128 take
    the merge engine) equal the C oracle's restatement of
    providers.py:266-301 (built from the same bit-identical sketches)."""
    g = pg.generate_kronecker(12, 16, 5)
    sk = pg.build_sketched_graph(g, "kmv", s=1.0, k_override=k)
    vals, lens = O.C.build_kmv(g.offsets, g.adjacency, k)
    assert np.array_equal(sk.values, vals) and np.array_equal(sk.lengths, lens)
    e = g.edges()
    p = pg.make_provider("kmv", sketched=sk)
    com, uni, want = O.C.pairs_kmv(vals, lens, k, np.diff(g.offsets), e[:, 0], e[:, 1])
    assert np.array_equal(p.pair_many(e[:, 0], e[:, 1]), want)
    c, u = p.pair_stats(e[:, 0], e[:, 1])
    assert np.array_equal(np.asarray(c), com) and np.array_equal(np.asarray(u), uni)
