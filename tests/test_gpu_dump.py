"""PGSKETCH v1 compatibility with the reference (tests/golden/pgsketch/*.bin,
written by the reference's dump_sketches; make_golden_dump.py): sketches
built on the device and dumped by this package are byte-identical, and the
reference's files load back to the same arrays and estimates."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pgsketch")
CASES = {
    "bloom_576_3": dict(kind="bloom", s=1.0, b=3, bits_override=576, seed=11),
    "bloom_budget": dict(kind="bloom", s=0.5, b=2, seed=12),
    "khash_16": dict(kind="khash", s=1.0, k_override=16, seed=13),
    "onehash_8": dict(kind="onehash", s=1.0, k_override=8, seed=14),
    "kmv_8": dict(kind="kmv", s=1.0, k_override=8, seed=15),
}
EST = {"bloom": "bf_and", "khash": "khash", "onehash": "onehash", "kmv": "kmv"}


@pytest.mark.parametrize("name", sorted(CASES))
def test_dump_bytes_and_load_match_reference(tmp_path, name):
    import paper_2208_11469_b200 as pg
    kw = dict(CASES[name])
    kind = kw.pop("kind")
    g = pg.generate_kronecker(7, 8, 3)
    sk = pg.build_sketched_graph(g, kind, **kw)
    path = tmp_path / f"{name}.bin"
    pg.dump_sketches(sk, path)
    ref = os.path.join(DIR, f"{name}.bin")
    assert open(path, "rb").read() == open(ref, "rb").read()
    back = pg.load_sketches(ref)
    assert back.kind.value == kind and back.n == g.n
    for f in ("bit_matrix", "ones", "entries", "lengths", "values"):
        a, b = getattr(back, f), getattr(sk, f)
        assert (a is None) == (b is None), f
        if a is not None:
            assert np.array_equal(a, b), f
    assert pg.tc_estimate(g, back, EST[kind]) == pg.tc_estimate(g, sk, EST[kind])


def test_directed_dump_matches_reference(tmp_path):
    import paper_2208_11469_b200 as pg
    g = pg.generate_kronecker(7, 8, 3)
    view = pg.degree_order(g)
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=256, seed=16,
                                 source="directed", view=view)
    pg.dump_sketches(sk, tmp_path / "d.bin")
    assert open(tmp_path / "d.bin", "rb").read() == \
        open(os.path.join(DIR, "bloom_directed.bin"), "rb").read()
    back = pg.load_sketches(os.path.join(DIR, "bloom_directed.bin"))
    assert back.source == "directed"
    p = pg.make_provider("bf_and", sketched=back)
    assert pg.four_clique_count(view, p) == pg.four_clique_count(
        view, pg.make_provider("bf_and", sketched=sk))
