"""Scalar with_set and pair against values the reference computed
(tests/golden/make_golden_withset.py; reference providers.py:164-175,
234-241, 303-307 and pair_many's scalar form): the one-warp pg_with_set
kernel with pinned mapped staging, and the pinned one-slot pair path.
Every value must be identical (same IEEE expressions)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLDEN, "withset.json")) as fh:
        return json.load(fh)


def gnp(n, p, seed):
    rng = np.random.default_rng(seed)
    iu, iv = np.triu_indices(n, k=1)
    mask = rng.random(len(iu)) < p
    return np.stack([iu[mask], iv[mask]], axis=1)


@pytest.mark.parametrize("name", ["g200", "dense120"])
def test_with_set_and_pair(gold, name):
    import paper_2208_11469_b200 as pg
    rec = gold[name]
    g = pg.CsrGraph.from_edges(gnp(rec["n"], rec["p"], rec["seed"]), n=rec["n"])
    for key, r in rec.items():
        if not isinstance(r, dict):
            continue
        sk = pg.build_sketched_graph(g, r["skind"], s=1.0, seed=rec["seed"] + 7, **r["kw"])
        p = pg.make_provider(key.split("_")[0] if not key.startswith("bf") else key.rsplit("_", 1)[0],
                             sketched=sk)
        for w, row in zip(rec["ws"], r["with_set"]):
            for m, want in zip(rec["sets"], row):
                got = p.with_set(w, np.asarray(m, dtype=np.int64))
                assert got == want, (key, w, m[:8], got, want)
        for (u, v), want in zip(rec["pairs"], r["pair"]):
            assert p.pair(u, v) == want, (key, u, v)
        # scalar estimators over sketch objects (reference estimators.py)
        for (u, v), want in zip(rec["pairs"][:8], r["est"]):
            a, b = sk.sketch(u), sk.sketch(v)
            su, sv = int(sk.sizes[u]), int(sk.sizes[v])
            if r["skind"] == "bloom":
                got = [pg.est_intersection_bf_and(a, b), pg.est_intersection_bf_limit(a, b),
                       pg.est_intersection_bf_or(a, b, su, sv),
                       pg.est_intersection_bf_or(a, b, su, sv, clamp=False)]
            elif r["skind"] in ("khash", "onehash"):
                got = [pg.est_jaccard_minhash(a, b), pg.est_intersection_minhash(a, b, su, sv)]
            else:
                got = [pg.est_intersection_kmv(a, b, su, sv),
                       pg.est_intersection_kmv(a, b, su, sv, clamp=False)]
            assert [float(x) for x in got] == want, (key, u, v)
