"""Run-to-run reproducibility of the fp64 sums (reference mining.py:63-80:
_chunked_sum's result does not depend on the thread count).  Integer
statistics are exact by construction; the KMV triangle-count sum is fp64 and
is reduced from fixed-slot partials in a fixed order (PartialSums), so
repeated passes are bit-identical whatever the dynamic schedule did."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def graph():
    import paper_2208_11469_b200 as pg
    return pg.generate_kronecker(16, 16, 2)


@pytest.mark.parametrize("k", [32, 64, 40])
def test_kmv_tc_bit_identical(graph, k):
    """k = 32/64: rank-directory engine (dynamic chunks); k = 40: merge-path
    engine (static slices)."""
    import paper_2208_11469_b200 as pg
    sk = pg.build_sketched_graph(graph, "kmv", s=1.0, k_override=k)
    vals = [pg.tc_estimate(graph, sk, "kmv") for _ in range(4)]
    assert len(set(vals)) == 1, vals


def test_kmv_loaded_sketches_bit_identical(graph, tmp_path):
    """Sketches without rank rows (loaded from a dump) take the merge-path
    TC engine: same value as the device-built ones within 1e-12, and
    reproducible."""
    import paper_2208_11469_b200 as pg
    sk = pg.build_sketched_graph(graph, "kmv", s=1.0, k_override=64)
    path = tmp_path / "kmv.pgs"
    pg.dump_sketches(sk, str(path))
    lk = pg.load_sketches(str(path))
    a = [pg.tc_estimate(graph, lk, "kmv") for _ in range(3)]
    assert len(set(a)) == 1
    assert a[0] == pytest.approx(pg.tc_estimate(graph, sk, "kmv"), rel=1e-12)


def test_integer_histograms_identical(graph):
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200.mining import tc_counts
    sk = pg.build_sketched_graph(graph, "bloom", s=1.0, b=2, bits_override=2048)
    p = pg.make_provider("bf_and", sketched=sk)
    h = [tc_counts(p, graph.device()).cpu().numpy() for _ in range(3)]
    assert all(np.array_equal(h[0], x) for x in h[1:])
