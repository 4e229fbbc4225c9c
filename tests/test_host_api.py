"""Host-side logic of the drop-in API (no GPU): plans, hashing, graphs,
dump format, Jaccard threshold arithmetic.  Mirrors the reference's own
unit tests for these pieces (reference tests/test_sketches.py:12-52,
tests/test_hashing.py, tests/test_graphs.py)."""

import numpy as np
import pytest

import paper_2208_11469_b200 as pg
from paper_2208_11469_b200.sketches import BudgetPlan


def k4():
    return pg.CsrGraph.from_edges([(a, b) for a in range(4) for b in range(a + 1, 4)], n=4)


def test_hash_golden_values():
    fam = pg.HashFamily(base_seed=pg.DEFAULT_HASH_SEED, count=2)
    assert fam.seed(0) == 0x2D0A2CC335CD72A7
    assert fam.seed(1) == 0x95527B2E69B24CDF
    assert pg.hash_to_bit(fam, 0, 12345, 256) == 47
    assert pg.hash_to_bit(fam, 1, 12345, 256) == 178
    assert pg.hash_to_unit(fam, 0, 12345) == 0.3926770316358376
    fam7 = pg.HashFamily(base_seed=7, count=2)
    assert pg.hash_to_bit(fam7, 0, 0, 65536) == 15605
    assert pg.hash_to_unit(fam7, 1, 99) == 0.05072011188429145


def test_hash_contracts():
    fam = pg.HashFamily(base_seed=1, count=2)
    with pytest.raises(IndexError):
        pg.hash_to_bit(fam, 2, 5, 10)
    with pytest.raises(ValueError):
        pg.hash_to_bit(fam, 0, 5, 0)
    with pytest.raises(ValueError):
        pg.HashFamily(base_seed=1, count=0)
    with pytest.raises(ValueError):
        pg.HashFamily(base_seed=1, count=1, algorithm="sha1")
    seen = set()
    for base in range(200):
        seen.update(pg.HashFamily(base_seed=base, count=8).seeds_array().tolist())
    assert len(seen) == 200 * 8


def test_plan_arithmetic():
    plan = pg.plan_budget(k4(), "bloom", s=0.25, b=1)
    assert plan.bits_per_vertex == 64 and plan.total_bits == 256
    with pytest.raises(pg.BudgetError):
        pg.plan_budget(k4(), "bloom", s=0.0)
    with pytest.raises(pg.BudgetError):
        pg.plan_budget(k4(), "bloom", s=0.01)
    star = pg.CsrGraph.from_edges([(0, i) for i in range(1, 40)])
    with pytest.raises(pg.BudgetError):
        pg.plan_budget(star, "onehash", s=0.2)
    rng = np.random.default_rng(0)
    edges = set()
    while len(edges) < 10_000:
        u, v = rng.integers(0, 1000, size=2)
        if u != v:
            edges.add((min(u, v), max(u, v)))
    g = pg.CsrGraph.from_edges(sorted(edges), n=1000)
    p = pg.plan_budget(g, "khash", s=0.25)
    assert p.entries_per_vertex == 5 and p.hash_count == 5
    assert BudgetPlan.explicit("kmv", 10, k=4).hash_count == 1
    with pytest.raises(ValueError):
        BudgetPlan.explicit("bloom", 10, bits=100)


def test_graph_contract_and_degree_order():
    g = pg.CsrGraph.from_edges([(0, 1), (1, 0), (2, 2), (1, 2), (3, 1)], n=5)
    assert g.m == 3 and g.self_loops_dropped == 1 and g.duplicates_dropped == 1
    g.validate()
    assert g.edges().tolist() == [[0, 1], [1, 2], [1, 3]]
    v = pg.degree_order(g)
    assert v.out_degrees().sum() == g.m
    for a in range(g.n):  # each edge oriented from lower to higher (deg, id)
        for b in v.out_neighbors(a):
            assert (g.degree(a), a) < (g.degree(b), b)


def test_generators_deterministic():
    a = pg.generate_kronecker(10, 8, 3)
    b = pg.generate_kronecker(10, 8, 3)
    assert np.array_equal(a.adjacency, b.adjacency)
    a.validate()
    er = pg.generate_erdos_renyi_gnm(500, 2000, 1)
    assert er.m == 2000
    er.validate()
    cl = pg.generate_chung_lu(4096, 16, 2.1, 3)
    cl.validate()
    d = cl.degrees()
    assert d[:16].mean() > 4 * d.mean()  # heavy head


def test_dump_load_roundtrip_host(tmp_path):
    fam = pg.HashFamily(base_seed=42, count=2)
    plan = BudgetPlan.explicit("bloom", 3, bits=128, b=2)
    rows = np.arange(6, dtype=np.uint64).reshape(3, 2) * np.uint64(0x0101010101010101)
    sg = pg.SketchedGraph("bloom", plan, fam, "undirected", [1, 2, 1], bit_matrix=rows,
                          ones=np.bitwise_count(rows).sum(axis=1).astype(np.int64))
    pg.dump_sketches(sg, tmp_path / "a.bin")
    back = pg.load_sketches(tmp_path / "a.bin")
    assert back.plan == sg.plan and back.seed == 42
    assert np.array_equal(back.bit_matrix, rows)
    plan_k = BudgetPlan.explicit("kmv", 2, k=3)
    vals = np.array([[0.1, 0.2, np.inf], [0.3, np.inf, np.inf]])
    sk = pg.SketchedGraph("kmv", plan_k, pg.HashFamily(1, 1), "directed", [2, 1],
                          values=vals, lengths=np.array([2, 1]))
    pg.dump_sketches(sk, tmp_path / "b.bin")
    back = pg.load_sketches(tmp_path / "b.bin")
    assert back.source == "directed" and np.array_equal(back.values, vals)
    assert back.sketch(0).hashes.tolist() == [0.1, 0.2]
    (tmp_path / "junk").write_bytes(b"not a sketch dump at all" * 4)
    with pytest.raises(ValueError):
        pg.load_sketches(tmp_path / "junk")


def test_jaccard_threshold_fp32():
    from paper_2208_11469_b200.mining import jaccard_min_matches
    assert jaccard_min_matches(32, 0.1) == 4
    for k in (1, 7, 32, 64, 100):
        for tau in (0.0, 0.05, 0.1, 0.5, 1.0):
            m = jaccard_min_matches(k, tau)
            assert all((np.float32(x) / np.float32(k) >= np.float32(tau)) == (x >= m)
                       for x in range(k + 1))


def test_swamidass_table_matches_scalar_formula():
    t = pg.swamidass_table(1024, 2)
    assert t[0] == 0.0
    assert t[1023] == pg.swamidass_value(1024, 2, 1023)
    assert t[1024] == t[1023]  # saturation fix
    assert pg.swamidass_value(2, 1, 1) == pytest.approx(2 * np.log(2), rel=1e-12)


def test_edge_range_partition():
    from paper_2208_11469_b200.sharding import edge_range, weighted_edge_range
    for m in (0, 1, 7, 1000, 15702278):
        for w in (1, 2, 3, 8):
            parts = [edge_range(m, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == m
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            assert max(e - b for b, e in parts) - min(e - b for b, e in parts) <= 1
    pref = np.cumsum(np.array([5, 1, 1, 1, 5, 1, 1, 1]))
    parts = [weighted_edge_range(pref, r, 2) for r in range(2)]
    assert parts[0][0] == 0 and parts[1][1] == 8 and parts[0][1] == parts[1][0]
