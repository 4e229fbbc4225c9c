"""Sampling TC baselines on the device vs the reference
(tests/golden/baselines.json from make_golden_baselines.py): the samples are
the reference's own numpy draws and the counts exact, so the values are
identical."""

import json
import os

import pytest

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                   "golden", "baselines.json")))


def _graph(pg, name):
    if name == "rmat12":
        return pg.generate_kronecker(12, 16, 8)
    return pg.generate_erdos_renyi_gnm(2000, 30000, 9)


@pytest.mark.parametrize("name", sorted(GOLD))
def test_doulion_and_reduced_execution(name):
    import paper_2208_11469_b200 as pg
    rec = GOLD[name]
    g = _graph(pg, name)
    assert (g.n, g.m) == (rec["n"], rec["m"])
    for key, want in rec["doulion"].items():
        p, seed = key.split("/")
        assert pg.doulion_tc(g, float(p), int(seed)) == want, key
    view = pg.degree_order(g)
    for key, want in rec["reduced"].items():
        f, seed = key.split("/")
        assert pg.reduced_execution_tc(view, float(f), int(seed)) == want, key
    with pytest.raises(ValueError):
        pg.doulion_tc(g, 0.0, 1)
    with pytest.raises(ValueError):
        pg.reduced_execution_tc(view, 1.5, 1)
