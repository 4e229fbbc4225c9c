"""Degree-oriented, hub-cached Bloom TC (pg_tc_bloom_hub) against the
ID-oriented kernel (pg_tc_bloom) and the C oracle: the same per-edge
popcounts (providers.py:150-162) over a different edge schedule, so the
histograms -- and with them every BF estimate -- must be identical
integers, for any number of staged hub rows and any shard split."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    import paper_2208_11469_b200 as pg
    return pg


def _hist(p, dev, monkeypatch, hub: bool, hubs=None):
    from paper_2208_11469_b200.mining import tc_counts
    monkeypatch.setenv("PG_TC_HUB", "1" if hub else "0")
    if hubs is None:
        monkeypatch.delenv("PG_TC_HUBS", raising=False)
    else:
        monkeypatch.setenv("PG_TC_HUBS", str(hubs))
    return tc_counts(p, dev).cpu().numpy()


@pytest.mark.parametrize("kind", ["bf_and", "bf_l", "bf_or"])
def test_hub_equals_id_oriented_rmat(pg, kind, monkeypatch):
    g = pg.generate_kronecker(16, 16, 5)
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048)
    p = pg.make_provider(kind, sketched=sk)
    dev = g.device()
    want = _hist(p, dev, monkeypatch, hub=False)
    for hubs in (None, 0, 1, 37, 500):
        got = _hist(p, dev, monkeypatch, hub=True, hubs=hubs)
        assert np.array_equal(got, want), hubs
    monkeypatch.setenv("PG_TC_HUB", "1")
    lay = p._tc_layout(dev)
    assert lay.kind == "hub" and lay.n_hubs == 500


def test_hub_histogram_vs_oracle(pg, monkeypatch):
    """Full AND-popcount histogram over every edge equals the C oracle's."""
    g = pg.generate_kronecker(15, 16, 9)
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048)
    p = pg.make_provider("bf_and", sketched=sk)
    got = _hist(p, g.device(), monkeypatch, hub=True)
    us, vs = O.upper_edges(g.offsets, g.adjacency)
    pop = O.C.pairs_bloom(sk.bit_matrix, 2048, False, us, vs)
    want = np.bincount(pop, minlength=2049)
    assert np.array_equal(got[:-1], want)


def test_hub_layout_every_edge_once(pg):
    """The hub slots name every undirected edge exactly once."""
    g = pg.generate_kronecker(12, 8, 3)
    dev = g.device()
    ug, vs, slots, hub_ids = dev.hub_slots(8, 50)
    ug = np.repeat(ug.cpu().numpy(), 8)[:slots]
    vs = vs.cpu().numpy()
    hub_ids = hub_ids.cpu().numpy()
    real = vs != -1
    v = np.where(vs <= -2, hub_ids[np.clip(-2 - vs, 0, None)], vs)
    u, v = ug[real], v[real]
    got = np.sort(np.minimum(u, v).astype(np.int64) * g.n + np.maximum(u, v))
    e = g.edges()
    want = np.sort(e[:, 0] * g.n + e[:, 1])
    assert np.array_equal(got, want)
    # orientation: low -> high (degree, ID) rank
    deg = g.degrees()
    key = lambda x: deg[x].astype(np.int64) * g.n + x  # noqa: E731
    assert np.all(key(u) < key(v))


def test_hub_sharded_ranges_sum(pg, monkeypatch):
    """Shard ranges of the hub layout (multiples of 32 slots) add up."""
    from paper_2208_11469_b200.mining import tc_counts
    monkeypatch.setenv("PG_TC_HUB", "1")
    g = pg.generate_kronecker(14, 16, 2)
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048)
    p = pg.make_provider("bf_and", sketched=sk)
    dev = g.device()
    whole = tc_counts(p, dev).cpu().numpy()
    parts = sum(tc_counts(p, dev, r, 3).cpu().numpy() for r in range(3))
    assert np.array_equal(parts, whole)


@pytest.mark.parametrize("bits", [512, 1024, 2048])
@pytest.mark.parametrize("kind", ["bf_and", "bf_l", "bf_or"])
def test_degree_orientation_equals_id_orientation(pg, bits, kind, monkeypatch):
    """The degree-oriented schedule of the wide engine (default) against
    the ID-oriented one: identical histograms (and BF_OR sums)."""
    from paper_2208_11469_b200.mining import tc_counts
    g = pg.generate_kronecker(15, 16, 6)
    sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=bits)
    p = pg.make_provider(kind, sketched=sk)
    dev = g.device()
    monkeypatch.setenv("PG_TC_HUB", "0")
    monkeypatch.setenv("PG_TC_ORIENT", "id")
    want = tc_counts(p, dev).cpu().numpy()
    monkeypatch.setenv("PG_TC_ORIENT", "degree")
    lay = p._tc_layout(dev)
    assert lay.kind == "degree"
    got = tc_counts(p, dev).cpu().numpy()
    assert np.array_equal(got, want)
    parts = sum(tc_counts(p, dev, r, 4).cpu().numpy() for r in range(4))
    assert np.array_equal(parts, want)
