"""4-clique counts with k-Hash / 1-Hash / KMV providers and with an exact
provider bound to another CSR, on the device (pg_4clique_sketch,
pg_4clique_exact_rows) vs values the reference computed
(tests/golden/make_golden_c4sketch.py: mining.py:133-154 with
MinHashProvider / KmvProvider.with_set, providers.py:234-241, 303-307, and
ExactProvider.for_graph, :117-118).

The per-triple estimates are fp64 and summed in a different order than the
reference's sequential loop, so sums agree to 1e-12 relative (north-star
tolerance 1e-6); the exact count and the triple counts are integers.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, KS, SMALL_NAMES, SMALL_SEEDS, small_graph

pytestmark = pytest.mark.gpu

RTOL = 1e-12


@pytest.fixture(scope="module")
def pg():
    import paper_2208_11469_b200 as pg
    return pg


@pytest.fixture(scope="module")
def c4g():
    with open(os.path.join(GOLDEN, "c4sketch.json")) as fh:
        return json.load(fh)


@pytest.fixture(params=["shared", "global"])
def cap_mode(request, monkeypatch):
    """'global': PG_C4S_CAP=4 drives every out-list longer than 4 through
    the per-warp global-scratch path (the path hub lists take)."""
    if request.param == "global":
        monkeypatch.setenv("PG_C4S_CAP", "4")
    else:
        monkeypatch.delenv("PG_C4S_CAP", raising=False)
    return request.param


@pytest.mark.parametrize("name", SMALL_NAMES)
@pytest.mark.parametrize("kind", ["khash", "onehash", "kmv"])
def test_small_directed(pg, small_golden, c4g, cap_mode, name, kind):
    g = small_graph(small_golden, name)
    view = pg.degree_order(g)
    rec = c4g["small"][name]
    for k in KS:
        dsk = pg.build_sketched_graph(g, kind, s=1.0, seed=SMALL_SEEDS[name] + 400, k_override=k,
                                      source="directed", view=view)
        got = pg.four_clique_count(view, pg.make_provider(kind, sketched=dsk))
        assert got == pytest.approx(rec[f"{kind}{k}_dir"], rel=RTOL, abs=1e-9), (kind, k)


@pytest.mark.parametrize("name", SMALL_NAMES)
@pytest.mark.parametrize("kind", ["khash", "onehash", "kmv"])
def test_small_undirected_sketches(pg, small_golden, c4g, name, kind):
    g = small_graph(small_golden, name)
    view = pg.degree_order(g)
    usk = pg.build_sketched_graph(g, kind, s=1.0, seed=SMALL_SEEDS[name] + 500, k_override=32)
    got = pg.four_clique_count(view, pg.make_provider(kind, sketched=usk))
    assert got == pytest.approx(c4g["small"][name][f"{kind}32_undir"], rel=RTOL, abs=1e-9)


@pytest.mark.parametrize("name", SMALL_NAMES)
def test_exact_for_graph(pg, small_golden, c4g, cap_mode, name):
    g = small_graph(small_golden, name)
    view = pg.degree_order(g)
    got = pg.four_clique_count(view, pg.make_provider("exact_merge", graph=g))
    assert got == c4g["small"][name]["exact_for_graph"]


@pytest.mark.parametrize("kind", ["khash", "onehash", "kmv"])
def test_rmat_s12(pg, c4g, cap_mode, kind):
    g = pg.generate_kronecker(12, 16, 4)
    view = pg.degree_order(g)
    rec = c4g["rmat"]["s12"]
    assert int(np.diff(view.offsets).max()) == rec["max_out_degree"]
    dsk = pg.build_sketched_graph(g, kind, s=1.0, k_override=16, source="directed", view=view)
    got = pg.four_clique_count(view, pg.make_provider(kind, sketched=dsk))
    assert got == pytest.approx(rec[f"{kind}16_dir"], rel=RTOL)


@pytest.mark.parametrize("kind", ["khash", "onehash", "kmv"])
def test_rmat_s16_sample(pg, c4g, kind):
    from paper_2208_11469_b200.mining import four_clique_sketch_sum
    g = pg.generate_kronecker(16, 16, 4)
    view = pg.degree_order(g)
    rec = c4g["rmat"]["s16_sample"]
    n_dir = int(view.offsets[-1])
    sample = np.sort(np.random.default_rng(0).choice(n_dir, size=n_dir // 100, replace=False))
    assert len(sample) == rec["sample_size"]
    dsk = pg.build_sketched_graph(g, kind, s=1.0, k_override=64, source="directed", view=view)
    total, trip = four_clique_sketch_sum(view, pg.make_provider(kind, sketched=dsk), sample)
    assert trip == rec["triples"]
    assert total == pytest.approx(rec[f"{kind}64_sum"], rel=RTOL)


def test_reproducible(pg):
    """Fixed reduction order and static schedule: bit-identical reruns."""
    g = pg.generate_kronecker(12, 16, 4)
    view = pg.degree_order(g)
    dsk = pg.build_sketched_graph(g, "kmv", s=1.0, k_override=16, source="directed", view=view)
    p = pg.make_provider("kmv", sketched=dsk)
    a = [pg.four_clique_count(view, p) for _ in range(3)]
    assert a[0] == a[1] == a[2]
