"""The plugin boundary with objects shaped like the reference's own.

Two routes a reference user takes:

1. the maintainer stub, ``integration/probgraph_b200.py``, executed here as
   ``probgraph.b200`` inside a stand-in ``probgraph`` package whose
   ``estimators.EstimatorKind`` is a separate enum class with the
   reference's values (estimators.py:54-63);
2. this package as the drop-in, handed graph / view / sketch objects that
   only carry the reference's field names (graphs.py:32-56,132-151;
   sketches.py:244-307) and enums of another class.

Inputs are the PGSKETCH files the reference wrote (tests/golden/pgsketch/),
parsed with this package's reader and re-wrapped in the reference-shaped
types below, so none of this package's graph/sketch classes reaches the API
under test; expected values are the reference's
own tc_estimate / pair_many / four_clique_count on those sketches
(expected.json, tests/golden/make_golden_dump.py).
"""

import dataclasses
import enum
import hashlib
import importlib.util
import json
import os
import sys
import types

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DIR = os.path.join(REPO, "tests", "golden", "pgsketch")
EXP = json.load(open(os.path.join(DIR, "expected.json")))


# ---- reference-shaped types (not this package's classes) -------------------
class RefSketchKind(str, enum.Enum):
    BLOOM = "bloom"
    KHASH = "khash"
    ONEHASH = "onehash"
    KMV = "kmv"


class RefEstimatorKind(str, enum.Enum):
    EXACT_MERGE = "exact_merge"
    EXACT_GALLOP = "exact_gallop"
    BF_AND = "bf_and"
    BF_L = "bf_l"
    BF_OR = "bf_or"
    KHASH = "khash"
    ONEHASH = "onehash"
    KMV = "kmv"


@dataclasses.dataclass(frozen=True)
class RefPlan:
    kind: RefSketchKind
    s: float
    bits_per_vertex: int
    entries_per_vertex: int
    hash_count: int
    total_bits: int
    budget_bits: int


@dataclasses.dataclass(frozen=True)
class RefFamily:
    base_seed: int
    count: int
    algorithm: str = "mix64"


class RefSketchedGraph:
    """Field names of reference SketchedGraph (sketches.py:244-307)."""

    def __init__(self, kind, plan, family, source, sizes, **arrays):
        self.kind, self.plan, self.family, self.source = kind, plan, family, source
        self.seed = family.base_seed
        self.sizes = np.asarray(sizes, dtype=np.int64)
        self.n = len(self.sizes)
        for f in ("bit_matrix", "ones", "entries", "lengths", "values"):
            setattr(self, f, arrays.get(f))

    capacity = property(lambda self: self.plan.entries_per_vertex)
    bit_length = property(lambda self: self.plan.bits_per_vertex)
    hash_count = property(lambda self: self.plan.hash_count)


class RefCsrGraph:
    def __init__(self, offsets, adjacency):
        self.offsets = np.asarray(offsets, dtype=np.int64)
        self.adjacency = np.asarray(adjacency, dtype=np.int64)
        self.n = len(self.offsets) - 1
        self.m = len(self.adjacency) // 2

    def degrees(self):
        return np.diff(self.offsets)

    def degree(self, v):
        return int(self.offsets[v + 1] - self.offsets[v])


def read_pgsketch(path) -> RefSketchedGraph:
    """A reference-written PGSKETCH v1 file (sketches.py:457-530) as a
    RefSketchedGraph (plain numpy arrays, foreign enum/plan/family types)."""
    import paper_2208_11469_b200 as pg
    ld = pg.load_sketches(path)  # parses the same bytes; re-wrapped below
    kind = RefSketchKind(ld.kind.value)
    p = ld.plan
    plan = RefPlan(kind, p.s, p.bits_per_vertex, p.entries_per_vertex, p.hash_count,
                   p.total_bits, p.budget_bits)
    fam = RefFamily(ld.family.base_seed, ld.family.count)
    arrays = {f: (None if getattr(ld, f) is None else np.array(getattr(ld, f)))
              for f in ("bit_matrix", "ones", "entries", "lengths", "values")}
    with open(path, "rb") as fh:
        assert fh.read(8).startswith(b"PGSKETCH")
    return RefSketchedGraph(kind, plan, fam, ld.source, ld.sizes.copy(), **arrays)


@pytest.fixture(scope="module")
def graph():
    import paper_2208_11469_b200 as pg
    g = pg.generate_kronecker(7, 8, 3)  # the graph make_golden_dump.py sketched
    assert g.m == EXP["m"]
    return RefCsrGraph(g.offsets, g.adjacency)


CASES = [("bloom_576_3", "bf_and"), ("bloom_576_3", "bf_l"), ("bloom_576_3", "bf_or"),
         ("bloom_budget", "bf_and"), ("bloom_budget", "bf_l"), ("bloom_budget", "bf_or"),
         ("khash_16", "khash"), ("onehash_8", "onehash"), ("kmv_8", "kmv")]


@pytest.mark.parametrize("name,kind", CASES)
def test_drop_in_accepts_reference_objects(graph, name, kind):
    import paper_2208_11469_b200 as pg
    sk = read_pgsketch(os.path.join(DIR, f"{name}.bin"))
    want = EXP[f"{name}/{kind}"]
    ek = RefEstimatorKind(kind)
    assert pg.tc_estimate(graph, sk, ek) == pytest.approx(want["tc_estimate"], rel=1e-12)
    p = pg.make_provider(ek, sketched=sk)
    e = np.stack([np.repeat(np.arange(graph.n), graph.degrees()), graph.adjacency], 1)
    e = e[e[:, 0] < e[:, 1]]
    pm = p.pair_many(e[:, 0], e[:, 1])
    assert hashlib.sha256(np.ascontiguousarray(pm, "<f8").tobytes()).hexdigest() == \
        want["pair_many_sha"]
    # the other entry points take the same objects
    jp = pg.jarvis_patrick_cluster(graph, p, 1.0)
    assert jp.singleton_count >= 0
    u, v = int(e[0, 0]), int(e[0, 1])
    assert np.isfinite(pg.vertex_similarity(u, v, "jaccard", p, graph))


def test_drop_in_four_clique_with_reference_view(graph):
    import paper_2208_11469_b200 as pg
    mine = pg.degree_order(pg.CsrGraph(graph.offsets, graph.adjacency))
    view = types.SimpleNamespace(n=mine.n, m=mine.m, rank=mine.rank.copy(),
                                 offsets=mine.offsets.copy(), adjacency=mine.adjacency.copy())
    sk = read_pgsketch(os.path.join(DIR, "bloom_directed.bin"))
    assert sk.source == "directed"
    p = pg.make_provider(RefEstimatorKind.BF_AND, sketched=sk)
    got = pg.four_clique_count(view, p)
    assert got == pytest.approx(EXP["bloom_directed/four_clique_count"], rel=1e-12)


def _load_stub():
    """integration/probgraph_b200.py as probgraph.b200 in a stand-in package."""
    from paper_2208_11469_b200 import _native
    from paper_2208_11469_b200.estimators import swamidass_value
    pkg = types.ModuleType("probgraph")
    pkg.__path__ = []
    est = types.ModuleType("probgraph.estimators")
    est.EstimatorKind = RefEstimatorKind
    est.swamidass_value = swamidass_value
    sys.modules["probgraph"] = pkg
    sys.modules["probgraph.estimators"] = est
    os.environ["PROBGRAPH_B200_LIB"] = _native.LIB_PATH
    spec = importlib.util.spec_from_file_location(
        "probgraph.b200", os.path.join(REPO, "integration", "probgraph_b200.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["probgraph.b200"] = mod
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("name,kind", [c for c in CASES if c[0].startswith("bloom")])
def test_maintainer_stub_matches_reference(graph, name, kind):
    stub = _load_stub()
    try:
        sk = read_pgsketch(os.path.join(DIR, f"{name}.bin"))
        got = stub.tc_estimate_b200(graph, sk, RefEstimatorKind(kind))
        assert got == pytest.approx(EXP[f"{name}/{kind}"]["tc_estimate"], rel=1e-12)
        with pytest.raises(ValueError):
            stub.tc_estimate_b200(graph, sk, RefEstimatorKind.KMV)
    finally:
        for k in ("probgraph", "probgraph.estimators", "probgraph.b200"):
            sys.modules.pop(k, None)
