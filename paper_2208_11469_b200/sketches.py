"""Sketch plans, per-set sketches and device-resident sketched graphs.

API restated from reference ``sketches.py``: ``SketchKind`` (:69-73),
``BudgetError`` (:76-77), ``BudgetPlan`` + ``explicit`` (:80-112),
``plan_budget`` (:115-138), the per-set sketch records (:145-184), the
per-set builders (:187-237), ``SketchedGraph`` (:244-307),
``build_sketched_graph`` (:399-451) and the PGSKETCH v1 dump format
(:457-530).

What differs is where the data lives: a :class:`SketchedGraph` built here
owns DEVICE tensors (HBM layouts in include/probgraph_b200.h) produced by the
sm_100a builders; the reference's host arrays (``bit_matrix``, ``ones``,
``entries``, ``lengths``, ``values``) are lazily materialised host mirrors
with the reference's dtypes (uint64 / int64 / float64), so user code and
``sketch(v)`` keep working.  A SketchedGraph constructed from host arrays
(e.g. ``load_sketches``) uploads them on first device use.
"""

from __future__ import annotations

import enum
import struct
from dataclasses import dataclass

import numpy as np

from .graphs import CsrGraph, DeviceCsr, DirectedView, degree_order
from .hashing import DEFAULT_HASH_SEED, HashFamily

__all__ = ["WORD_BITS", "SketchKind", "BudgetError", "BudgetPlan",
           "plan_budget", "BloomSketch", "KHashSketch", "OneHashSketch",
           "KmvSketch", "build_bloom", "build_khash", "build_onehash",
           "build_kmv", "SketchedGraph", "build_sketched_graph",
           "dump_sketches", "load_sketches", "as_sketched_graph"]

WORD_BITS = 64


class SketchKind(str, enum.Enum):
    BLOOM = "bloom"
    KHASH = "khash"
    ONEHASH = "onehash"
    KMV = "kmv"


class BudgetError(ValueError):
    """The storage budget cannot fit the minimum per-vertex sketch."""


@dataclass(frozen=True)
class BudgetPlan:
    kind: SketchKind
    s: float
    bits_per_vertex: int
    entries_per_vertex: int
    hash_count: int
    total_bits: int
    budget_bits: int

    @classmethod
    def explicit(cls, kind, n: int, *, bits: int = 0, k: int = 0,
                 b: int = 1) -> "BudgetPlan":
        kind = SketchKind(kind)
        if kind is SketchKind.BLOOM:
            if bits < WORD_BITS or bits % WORD_BITS:
                raise ValueError(
                    f"Bloom size must be a positive multiple of {WORD_BITS}")
            return cls(kind, 1.0, bits, 0, b, n * bits, n * bits)
        if k < 1:
            raise ValueError("k must be >= 1")
        total = n * k * WORD_BITS
        return cls(kind, 1.0, k * WORD_BITS, k,
                   k if kind is SketchKind.KHASH else 1, total, total)


def plan_budget(graph: CsrGraph, kind, s: float, b: int = 1) -> BudgetPlan:
    """Uniform per-vertex size for a fraction s of the (n + 2m)-word CSR."""
    kind = SketchKind(kind)
    if not 0 < s <= 1:
        raise BudgetError(f"storage budget s={s} outside (0, 1]")
    if graph.n == 0:
        raise BudgetError("cannot plan sketches for an empty graph")
    budget_bits = int(s * (graph.n + 2 * graph.m) * WORD_BITS)
    if kind is SketchKind.BLOOM:
        if b < 1:
            raise ValueError("need at least one hash function")
        bits = (budget_bits // graph.n) // WORD_BITS * WORD_BITS
        if bits < WORD_BITS:
            raise BudgetError(
                f"budget s={s} cannot fit one {WORD_BITS}-bit word per vertex")
        return BudgetPlan(kind, s, bits, 0, b, graph.n * bits, budget_bits)
    k = max(1, int(s * 2 * graph.m / graph.n))
    total = graph.n * k * WORD_BITS
    if total > budget_bits:
        raise BudgetError(
            f"budget s={s} cannot fit one {WORD_BITS}-bit entry per vertex")
    return BudgetPlan(kind, s, k * WORD_BITS, k,
                      k if kind is SketchKind.KHASH else 1, total, budget_bits)


# ---------------------------------------------------------------------------
# per-set sketches (host records, same fields as the reference)


@dataclass
class BloomSketch:
    words: np.ndarray
    bit_length: int
    hash_count: int
    ones: int
    seed: int = 0

    def recount(self) -> int:
        return int(np.bitwise_count(self.words).sum())

    def contains(self, family: HashFamily, key: int) -> bool:
        from .hashing import hash_to_bit
        for i in range(self.hash_count):
            pos = hash_to_bit(family, i, key, self.bit_length)
            if not (int(self.words[pos >> 6]) >> (pos & 63)) & 1:
                return False
        return True


@dataclass
class KHashSketch:
    entries: np.ndarray
    capacity: int
    seed: int = 0


@dataclass
class OneHashSketch:
    entries: np.ndarray
    capacity: int
    seed: int = 0


@dataclass
class KmvSketch:
    hashes: np.ndarray
    capacity: int
    seed: int = 0


def _single_row_sketch(neigh, kind: SketchKind, plan: BudgetPlan,
                       family: HashFamily) -> "SketchedGraph":
    """Sketch of one explicit set: a 1-vertex CSR through the device builder."""
    neigh = np.asarray(neigh, dtype=np.int64).reshape(-1)
    if len(neigh) and (neigh.min() < 0 or neigh.max() >= 2 ** 31):
        raise ValueError("set members must be int32 vertex IDs")
    members = np.unique(neigh)  # a set: sorted, duplicate free
    offsets = np.asarray([0, len(members)], dtype=np.int64)
    dev = DeviceCsr(offsets, members)
    return _build_on_device(dev, kind, plan, family, "undirected",
                            np.asarray([len(members)], dtype=np.int64))


def build_bloom(neigh, plan: BudgetPlan, family: HashFamily) -> BloomSketch:
    if plan.kind is not SketchKind.BLOOM:
        raise ValueError("plan is not a Bloom plan")
    sg = _single_row_sketch(neigh, SketchKind.BLOOM, plan, family)
    return BloomSketch(sg.bit_matrix[0], plan.bits_per_vertex, plan.hash_count,
                       int(sg.ones[0]), family.base_seed)


def _kplan(kind: SketchKind, k: int) -> BudgetPlan:
    if k < 1:
        raise ValueError("k must be >= 1")
    return BudgetPlan.explicit(kind, 1, k=k)


def build_khash(neigh, k: int, family: HashFamily) -> KHashSketch:
    plan = _kplan(SketchKind.KHASH, k)
    if len(np.asarray(neigh).reshape(-1)) == 0:
        return KHashSketch(np.empty(0, dtype=np.int64), k, family.base_seed)
    sg = _single_row_sketch(neigh, SketchKind.KHASH, plan, family)
    return KHashSketch(sg.entries[0].copy(), k, family.base_seed)


def build_onehash(neigh, k: int, family: HashFamily) -> OneHashSketch:
    plan = _kplan(SketchKind.ONEHASH, k)
    sg = _single_row_sketch(neigh, SketchKind.ONEHASH, plan, family)
    return OneHashSketch(sg.entries[0, :sg.lengths[0]].copy(), k,
                         family.base_seed)


def build_kmv(neigh, k: int, family: HashFamily) -> KmvSketch:
    plan = _kplan(SketchKind.KMV, k)
    sg = _single_row_sketch(neigh, SketchKind.KMV, plan, family)
    return KmvSketch(sg.values[0, :sg.lengths[0]].copy(), k, family.base_seed)


# ---------------------------------------------------------------------------
# whole-graph sketches


class SketchedGraph:
    """One sketch per vertex, resident in HBM, with lazy host mirrors."""

    def __init__(self, kind, plan: BudgetPlan, family: HashFamily,
                 source: str, sizes, *, bit_matrix=None, ones=None,
                 entries=None, lengths=None, values=None, device=None,
                 ready=None):
        self.kind = SketchKind(kind)
        self.plan = plan
        self.family = family
        self.seed = family.base_seed
        self.source = source
        # sizes may be given lazily as ("offsets", host_offsets): np.diff is
        # then only paid when a host caller asks for them
        if isinstance(sizes, tuple) and sizes and sizes[0] == "offsets":
            self._sizes = None
            self._sizes_from = sizes[1]
            self.n = len(sizes[1]) - 1
        else:
            self._sizes = np.asarray(sizes, dtype=np.int64)
            self._sizes_from = None
            self.n = len(self._sizes)
        self._host = {"bit_matrix": bit_matrix, "ones": ones,
                      "entries": entries, "lengths": lengths,
                      "values": values}
        self._dev = dict(device) if device else {}
        # CUDA event after which the device tensors are complete (builds on
        # a side stream); consumers' streams wait on it at access time
        self._ready = ready
        self._chunk_ready = []  # per upload chunk (v0, v1, copy event, build event)
        self._chunk_dev = None

    def _wait_ready(self) -> None:
        if self._ready is not None:
            import torch
            if torch.cuda.is_current_stream_capturing():
                # a capture cannot depend on an outside event: the build must
                # be complete (it is after any earlier eager use)
                self._ready.synchronize()
                return
            torch.cuda.current_stream().wait_event(self._ready)
            if self._ready.query():  # completed: later callers need no wait
                self._ready = None

    @property
    def sizes(self) -> np.ndarray:
        """int64 size of every sketched set (a CSR degree)."""
        if self._sizes is None:
            self._sizes = np.diff(np.asarray(self._sizes_from, dtype=np.int64))
        return self._sizes

    # -- plan shortcuts (reference :270-280)
    @property
    def capacity(self) -> int:
        return self.plan.entries_per_vertex

    @property
    def bit_length(self) -> int:
        return self.plan.bits_per_vertex

    @property
    def hash_count(self) -> int:
        return self.plan.hash_count

    # -- device side
    def device_tensors(self) -> dict:
        """Device buffers; uploads host arrays on first use if needed."""
        import torch
        from .graphs import _to_device
        self._wait_ready()
        d = self._dev
        if "sizes" not in d:
            d["sizes"] = _to_device(self.sizes, torch.int32)
        if "seeds" not in d:
            d["seeds"] = torch.from_numpy(
                self.family.seeds_array().view(np.int64)).cuda()
        h = self._host
        if self.kind is SketchKind.BLOOM and "rows" not in d:
            d["rows"] = _to_device(np.asarray(h["bit_matrix"], dtype=np.uint64)
                                   .view(np.int64), torch.int64)
            d["ones"] = _to_device(h["ones"], torch.int32)
        elif self.kind in (SketchKind.KHASH, SketchKind.ONEHASH) and "entries" not in d:
            d["entries"] = _to_device(h["entries"], torch.int32)
            if self.kind is SketchKind.ONEHASH:
                d["lengths"] = _to_device(h["lengths"], torch.int32)
        elif self.kind is SketchKind.KMV and "values" not in d:
            d["values"] = _to_device(h["values"], torch.float64)
            d["lengths"] = _to_device(h["lengths"], torch.int32)
        return d

    def _mirror(self, name: str):
        if self._host.get(name) is None and self._dev:
            t = self._dev.get({"bit_matrix": "rows"}.get(name, name))
            if t is None:
                return None
            self._wait_ready()
            a = t.cpu().numpy()
            if name == "bit_matrix":
                a = a.view(np.uint64)
            elif name == "values":
                a = a.astype(np.float64)
            else:
                a = a.astype(np.int64)
            self._host[name] = a
        return self._host.get(name)

    bit_matrix = property(lambda self: self._mirror("bit_matrix"))
    ones = property(lambda self: self._mirror("ones"))
    entries = property(lambda self: self._mirror("entries"))
    lengths = property(lambda self: self._mirror("lengths"))
    values = property(lambda self: self._mirror("values"))

    def _row(self, name: str, v: int):
        """Row v of a sketch array: from the host mirror when it exists,
        else one row copied from the device (a scalar call must not pull
        the whole matrix -- 4 GiB at config 5 -- to the host)."""
        h = self._host.get(name)
        if h is not None or not self._dev:
            return self._mirror(name)[v]
        t = self._dev.get({"bit_matrix": "rows"}.get(name, name))
        if t is None:
            return self._mirror(name)[v]
        self._wait_ready()
        a = t[int(v)].cpu().numpy()
        if name == "bit_matrix":
            return a.view(np.uint64)
        if name == "values":
            return a.astype(np.float64)
        return np.asarray(a, dtype=np.int64)

    def sketch(self, v: int):
        v = int(v)
        if v < 0:  # numpy row indexing, as the reference's self.bit_matrix[v]
            v += self.n
        if not 0 <= v < self.n:
            raise IndexError(f"index {v} is out of bounds for axis 0 with size {self.n}")
        if self.kind is SketchKind.BLOOM:
            return BloomSketch(self._row("bit_matrix", v), self.bit_length,
                               self.hash_count, int(self._row("ones", v)), self.seed)
        if self.kind is SketchKind.KHASH:
            row = self._row("entries", v)
            return KHashSketch(row if self.sizes[v] > 0 else row[:0],
                               self.capacity, self.seed)
        if self.kind is SketchKind.ONEHASH:
            return OneHashSketch(self._row("entries", v)[:int(self._row("lengths", v))],
                                 self.capacity, self.seed)
        return KmvSketch(self._row("values", v)[:int(self._row("lengths", v))],
                         self.capacity, self.seed)

    def extra_bits_used(self) -> int:
        if self.kind is SketchKind.BLOOM:
            return self.n * self.bit_length
        if self.kind is SketchKind.KHASH:
            return int(np.count_nonzero(self.sizes > 0)) * self.capacity * WORD_BITS
        return int(self.lengths.sum()) * WORD_BITS

    def extra_bytes_used(self) -> int:
        return self.extra_bits_used() // 8


def as_sketched_graph(obj) -> SketchedGraph:
    """This package's SketchedGraph for any object exposing the reference
    SketchedGraph fields (sketches.py:244-307: kind, plan, family, source,
    sizes and the kind's bit_matrix/ones, entries(/lengths) or
    values/lengths host arrays) -- e.g. sketches built or loaded by the
    reference itself.  Enums are matched by value, the arrays are uploaded
    on first device use, and the wrapper is cached on the object."""
    if isinstance(obj, SketchedGraph):
        return obj
    from .graphs import _ADOPTED
    cached = _ADOPTED.get(id(obj))
    if cached is not None and cached[0] is obj:
        return cached[1]
    try:
        kind = SketchKind(getattr(obj.kind, "value", obj.kind))
        p, fam = obj.plan, obj.family
        plan = BudgetPlan(kind, float(p.s), int(p.bits_per_vertex), int(p.entries_per_vertex),
                          int(p.hash_count), int(p.total_bits), int(p.budget_bits))
        family = HashFamily(int(fam.base_seed), int(fam.count),
                            getattr(fam, "algorithm", "mix64"))
        source = str(getattr(obj.source, "value", obj.source))
        sizes = np.asarray(obj.sizes, dtype=np.int64)
    except AttributeError as exc:
        raise TypeError(f"expected a SketchedGraph: {exc}") from None

    def arr(name):
        a = getattr(obj, name, None)
        return None if a is None else np.asarray(a)

    sg = SketchedGraph(kind, plan, family, source, sizes, bit_matrix=arr("bit_matrix"),
                       ones=arr("ones"), entries=arr("entries"), lengths=arr("lengths"),
                       values=arr("values"))
    _ADOPTED[id(obj)] = (obj, sg)
    return sg


def _launch_builders(dev: DeviceCsr, kind: SketchKind, plan: BudgetPlan, seeds, out,
                     v0: int, v1: int, stream: int) -> None:
    """Build the sketches of vertices [v0, v1) into the rows of `out`."""
    from . import _native as N
    n = v1 - v0
    if n <= 0:
        return
    off = N.ptr(dev.offsets) + 8 * v0  # offsets stay absolute into adj

    def row(t):
        return N.ptr(t) + v0 * t.stride(0) * t.element_size()

    if kind is SketchKind.BLOOM:
        N.call("pg_build_bloom", off, N.ptr(dev.adj), n, plan.bits_per_vertex,
               plan.hash_count, N.ptr(seeds), row(out["rows"]), row(out["ones"]), stream)
        return
    k = plan.entries_per_vertex
    if kind is SketchKind.KHASH:
        N.call("pg_build_khash", off, N.ptr(dev.adj), n, k, N.ptr(seeds),
               row(out["entries"]), stream)
    elif kind is SketchKind.ONEHASH:
        N.call("pg_build_onehash", off, N.ptr(dev.adj), n, k, N.ptr(seeds),
               row(out["entries"]), row(out["lengths"]), stream)
    else:
        # values plus their global-rank rows (the KMV TC engine's layout)
        N.call("pg_build_kmv_ranked", off, N.ptr(dev.adj), n, k, N.ptr(seeds),
               N.ptr(out["rank_of"]), N.ptr(out["rank_values"]),
               row(out["values"]), row(out["ranks"]), row(out["lengths"]), stream)


def _alloc_outputs(kind: SketchKind, plan: BudgetPlan, n: int) -> dict:
    import torch
    alloc_n = max(n, 1)
    if kind is SketchKind.BLOOM:
        words = plan.bits_per_vertex // WORD_BITS
        return {"rows": torch.empty((alloc_n, words), dtype=torch.int64, device="cuda"),
                "ones": torch.empty(alloc_n, dtype=torch.int32, device="cuda")}
    k = plan.entries_per_vertex
    if kind is SketchKind.KHASH:
        return {"entries": torch.empty((alloc_n, k), dtype=torch.int32, device="cuda")}
    if kind is SketchKind.ONEHASH:
        return {"entries": torch.empty((alloc_n, k), dtype=torch.int32, device="cuda"),
                "lengths": torch.empty(alloc_n, dtype=torch.int32, device="cuda")}
    return {"values": torch.empty((alloc_n, k), dtype=torch.float64, device="cuda"),
            "ranks": torch.empty((alloc_n, k), dtype=torch.int32, device="cuda"),
            "rank_of": torch.empty(alloc_n, dtype=torch.int32, device="cuda"),
            "rank_values": torch.empty(alloc_n, dtype=torch.float64, device="cuda"),
            "lengths": torch.empty(alloc_n, dtype=torch.int32, device="cuda")}


def _prepare_builders(kind: SketchKind, n: int, seeds, out, stream: int) -> None:
    """Whole-graph tables the per-chunk builders read (KMV value ranks)."""
    from . import _native as N
    if kind is SketchKind.KMV:
        N.call("pg_kmv_rank_table", n, N.ptr(seeds), N.ptr(out["rank_of"]),
               N.ptr(out["rank_values"]), stream)


def _build_on_device(dev: DeviceCsr, kind: SketchKind, plan: BudgetPlan,
                     family: HashFamily, source: str,
                     sizes: np.ndarray) -> SketchedGraph:
    """Launch the builders on the device.  If the CSR upload is still in
    flight in chunks (DeviceCsr.upload_chunks), build each chunk on a side
    stream as soon as it lands, overlapping the H2D copy with the build; the
    result then carries a readiness event (SketchedGraph._wait_ready)."""
    import torch
    from . import _native as N
    from .graphs import side_stream
    n = dev.n

    def device_seeds(stream):
        # derived on the device: a host copy would queue behind the CSR upload
        seeds = torch.empty(family.count, dtype=torch.int64, device="cuda")
        N.call("pg_family_seeds_device", family.base_seed, family.count, N.ptr(seeds), stream)
        return seeds

    chunks = dev.take_upload_chunks()
    if chunks:
        cur = torch.cuda.current_stream()
        bs = side_stream("build")
        with torch.cuda.stream(bs):  # allocations ordered on bs
            seeds = device_seeds(bs.cuda_stream)
            out = _alloc_outputs(kind, plan, n)
            _prepare_builders(kind, n, seeds, out, bs.cuda_stream)
            chunk_ready = []
            for v0, v1, ev in chunks:
                bs.wait_event(ev)
                _launch_builders(dev, kind, plan, seeds, out, v0, v1, bs.cuda_stream)
                built = torch.cuda.Event()
                built.record(bs)
                # (copy event, build event): a consumer may start on the
                # vertex range once both passed (mining.tc_counts)
                chunk_ready.append((v0, v1, ev, built))
            ready = torch.cuda.Event()
            ready.record(bs)
        # consumers wait for `ready` when they touch the sketches
        # (SketchedGraph._wait_ready), so work that only needs the CSR -- the
        # edge-slot layout -- overlaps the last chunks' build
        seeds.record_stream(cur)
        for t in out.values():
            t.record_stream(cur)
    else:
        ready = None
        chunk_ready = []
        seeds = device_seeds(N.stream_handle())
        out = _alloc_outputs(kind, plan, n)
        _prepare_builders(kind, n, seeds, out, N.stream_handle())
        _launch_builders(dev, kind, plan, seeds, out, 0, n, N.stream_handle())
    out = {key: t[:n] for key, t in out.items()}
    out.update(seeds=seeds, sizes=dev.degrees)
    sg = SketchedGraph(kind, plan, family, source, sizes, device=out, ready=ready)
    sg._chunk_ready = chunk_ready
    sg._chunk_dev = dev if chunk_ready else None
    return sg


def build_sketched_graph(graph: CsrGraph, kind, s: float, b: int = 1,
                         seed: int = DEFAULT_HASH_SEED, *,
                         source: str = "undirected",
                         view: DirectedView | None = None,
                         k_override: int | None = None,
                         bits_override: int | None = None) -> SketchedGraph:
    """Sketch every neighbourhood on the device (reference :399-451)."""
    from .graphs import as_csr_graph, as_directed_view
    graph = as_csr_graph(graph)
    if view is not None:
        view = as_directed_view(view)
    kind = SketchKind(getattr(kind, "value", kind))
    if source == "undirected":
        host_off, dev_src = graph.offsets, graph
    elif source == "directed":
        if view is None:
            view = degree_order(graph)
        host_off, dev_src = view.offsets, view
    else:
        raise ValueError("source must be 'undirected' or 'directed'")
    sizes = ("offsets", host_off)  # materialised lazily (SketchedGraph.sizes)
    if kind is SketchKind.BLOOM and bits_override is not None:
        plan = BudgetPlan.explicit(kind, graph.n, bits=bits_override, b=b)
    elif kind is not SketchKind.BLOOM and k_override is not None:
        plan = BudgetPlan.explicit(kind, graph.n, k=k_override)
    else:
        plan = plan_budget(graph, kind, s, b)
    family = HashFamily(base_seed=seed, count=plan.hash_count)
    return _build_on_device(dev_src.device(), kind, plan, family, source, sizes)


# ---------------------------------------------------------------------------
# PGSKETCH v1 dump / restore (reference :457-530)

_MAGIC = b"PGSKETCH"
_VERSION = 1
_HEADER = "<8sHBBIQQQdQQ"
_KIND_CODE = {SketchKind.BLOOM: 0, SketchKind.KHASH: 1, SketchKind.ONEHASH: 2,
              SketchKind.KMV: 3}
_SOURCE_CODE = {"undirected": 0, "directed": 1}


def dump_sketches(sg: SketchedGraph, path) -> None:
    param = sg.bit_length if sg.kind is SketchKind.BLOOM else sg.capacity
    head = struct.pack(_HEADER, _MAGIC, _VERSION, _KIND_CODE[sg.kind],
                       _SOURCE_CODE[sg.source], sg.plan.hash_count, sg.n, param,
                       sg.seed, sg.plan.s, sg.plan.total_bits,
                       sg.plan.budget_bits)
    arrays = [sg.sizes.astype("<i8")]
    if sg.kind is SketchKind.BLOOM:
        arrays += [sg.ones.astype("<i8"), sg.bit_matrix.astype("<u8")]
    elif sg.kind is SketchKind.KHASH:
        arrays += [sg.entries.astype("<i8")]
    elif sg.kind is SketchKind.ONEHASH:
        arrays += [sg.lengths.astype("<i8"), sg.entries.astype("<i8")]
    else:
        arrays += [sg.lengths.astype("<i8"), sg.values.astype("<f8")]
    with open(path, "wb") as fh:
        fh.write(head)
        for a in arrays:
            fh.write(np.ascontiguousarray(a).tobytes())


def load_sketches(path) -> SketchedGraph:
    with open(path, "rb") as fh:
        raw = fh.read(struct.calcsize(_HEADER))
        if len(raw) < struct.calcsize(_HEADER):
            raise ValueError("not a sketch dump")
        (magic, version, kcode, scode, hash_count, n, param, seed, s,
         total_bits, budget_bits) = struct.unpack(_HEADER, raw)
        if magic != _MAGIC:
            raise ValueError("not a sketch dump")
        if version != _VERSION:
            raise ValueError(f"unsupported sketch dump version {version}")
        kind = {v: k for k, v in _KIND_CODE.items()}[kcode]
        source = {v: k for k, v in _SOURCE_CODE.items()}[scode]

        def read(dtype, count):
            return np.frombuffer(fh.read(8 * count), dtype=dtype).copy()

        sizes = read("<i8", n).astype(np.int64)
        family = HashFamily(base_seed=seed, count=hash_count)
        if kind is SketchKind.BLOOM:
            plan = BudgetPlan(kind, s, param, 0, hash_count, total_bits,
                              budget_bits)
            ones = read("<i8", n).astype(np.int64)
            wpr = param // WORD_BITS
            mat = read("<u8", n * wpr).astype(np.uint64).reshape(n, wpr)
            return SketchedGraph(kind, plan, family, source, sizes,
                                 bit_matrix=mat, ones=ones)
        plan = BudgetPlan(kind, s, param * WORD_BITS, param, hash_count,
                          total_bits, budget_bits)
        if kind is SketchKind.KHASH:
            ent = read("<i8", n * param).astype(np.int64).reshape(n, param)
            return SketchedGraph(kind, plan, family, source, sizes, entries=ent)
        lengths = read("<i8", n).astype(np.int64)
        if kind is SketchKind.ONEHASH:
            ent = read("<i8", n * param).astype(np.int64).reshape(n, param)
            return SketchedGraph(kind, plan, family, source, sizes,
                                 entries=ent, lengths=lengths)
        vals = read("<f8", n * param).astype(np.float64).reshape(n, param)
        return SketchedGraph(kind, plan, family, source, sizes, values=vals,
                             lengths=lengths)
