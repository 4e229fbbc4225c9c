"""Sketch sizes beyond the tuned kernels: Bloom rows of 40,000 / 65,600 /
70,016 bits (generic TC histogram above 32,768 bits, generic builder above
65,536, generic 4-clique above 16,384) and k = 300 / 513 (generic builders
and estimators above 256), vs values the reference computed
(tests/golden/make_golden_generic.py; reference sketches.py:115-138 gives
such sizes on dense graphs).  Sketch arrays and per-edge estimates are
compared by sha256 of their canonical bytes (bit-exact); sums to 1e-12."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

RTOL = 1e-12


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def gen():
    with open(os.path.join(GOLDEN, "generic.json")) as fh:
        return json.load(fh)


def gnp(n, p, seed):
    rng = np.random.default_rng(seed)
    iu, iv = np.triu_indices(n, k=1)
    mask = rng.random(len(iu)) < p
    return np.stack([iu[mask], iv[mask]], axis=1)


@pytest.fixture(scope="module")
def dense(gen):
    import paper_2208_11469_b200 as pg
    r = gen["dense300"]
    g = pg.CsrGraph.from_edges(gnp(r["n"], r["p"], r["seed"]), n=r["n"])
    assert g.m == r["m"]
    return g


def canon_sha(sk):
    out = {}
    if sk.kind.value == "bloom":
        out["bit_matrix"] = sha(sk.bit_matrix.astype("<u8"))
        out["ones"] = sha(sk.ones.astype("<i8"))
    elif sk.kind.value in ("khash", "onehash"):
        out["entries"] = sha(sk.entries.astype("<i8"))
        if sk.kind.value == "onehash":
            out["lengths"] = sha(sk.lengths.astype("<i8"))
    else:
        out["values"] = sha(sk.values.astype("<f8"))
        out["lengths"] = sha(sk.lengths.astype("<i8"))
    return out


@pytest.mark.parametrize("bits,b", [(40000, 2), (70016, 2), (65600, 1)])
def test_wide_bloom(gen, dense, bits, b):
    import paper_2208_11469_b200 as pg
    rec = gen["dense300"][f"bloom{bits}_{b}"]
    sk = pg.build_sketched_graph(dense, "bloom", s=1.0, b=b, bits_override=bits)
    for k2, v2 in canon_sha(sk).items():
        assert v2 == rec[k2], k2
    e = dense.edges()
    for kind in ("bf_and", "bf_l", "bf_or"):
        p = pg.make_provider(kind, sketched=sk)
        assert sha(p.pair_many(e[:, 0], e[:, 1]).astype("<f8")) == rec[f"pairs_{kind}"], kind
        assert pg.tc_estimate(dense, sk, kind) == pytest.approx(rec[f"tc_{kind}"], rel=RTOL), kind


@pytest.mark.parametrize("k", [300, 513])
@pytest.mark.parametrize("kind", ["khash", "onehash", "kmv"])
def test_large_k(gen, dense, kind, k):
    import paper_2208_11469_b200 as pg
    rec = gen["dense300"][f"{kind}{k}"]
    sk = pg.build_sketched_graph(dense, kind, s=1.0, k_override=k)
    for k2, v2 in canon_sha(sk).items():
        assert v2 == rec[k2], k2
    p = pg.make_provider(kind, sketched=sk)
    e = dense.edges()
    assert sha(p.pair_many(e[:, 0], e[:, 1]).astype("<f8")) == rec["pairs"]
    assert pg.tc_estimate(dense, sk, kind) == pytest.approx(rec["tc"], rel=RTOL)
    jp = pg.jarvis_patrick_cluster(dense, p, 50.0)
    assert [len(jp.kept_edges), jp.cluster_count, jp.singleton_count] == rec["jp50"]
    if kind == "khash":
        jc = pg.jaccard_cluster_count(dense, sk, 0.1)
        assert jc.kept_hat == rec["kept_jhat_ge_0.1"]
        assert jc.kept_similarity == rec["kept_sim_ge_0.1"]


@pytest.mark.parametrize("kind,k", [("khash", 300), ("onehash", 300), ("kmv", 300), ("onehash", 40),
                                    ("kmv", 40)])
def test_4clique_large_k(gen, kind, k):
    import paper_2208_11469_b200 as pg
    r = gen["c4g120"]
    g = pg.CsrGraph.from_edges(gnp(r["n"], r["p"], r["seed"]), n=r["n"])
    view = pg.degree_order(g)
    dsk = pg.build_sketched_graph(g, kind, s=1.0, k_override=k, source="directed", view=view)
    got = pg.four_clique_count(view, pg.make_provider(kind, sketched=dsk))
    assert got == pytest.approx(r[f"{kind}{k}_dir"], rel=RTOL)


@pytest.mark.parametrize("bits", [70016, 20032])
def test_4clique_wide_bloom(gen, bits):
    import paper_2208_11469_b200 as pg
    r = gen["c4g120"]
    g = pg.CsrGraph.from_edges(gnp(r["n"], r["p"], r["seed"]), n=r["n"])
    view = pg.degree_order(g)
    dsk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=bits, source="directed",
                                  view=view)
    for kind in ("bf_and", "bf_or"):
        got = pg.four_clique_count(view, pg.make_provider(kind, sketched=dsk))
        assert got == pytest.approx(r[f"bloom{bits}_{kind}_dir"], rel=RTOL), kind
