"""CSR graphs: the input contract of the engine, plus seeded generators.

Host arrays follow the reference contract exactly (reference graphs.py:32-166:
int64 ``offsets``/``adjacency``, sorted symmetric loop-free rows, ``edges()``
yielding u < v in CSR order, ``degree_order`` ranking by (degree, id)).  The
device mirror (:class:`DeviceCsr`) narrows the adjacency to int32 and keeps
int64 offsets; it is built once per graph and cached.

Generators (input preparation, outside every timed region):
  * ``generate_kronecker`` -- R-MAT with the reference's initiator and draw
    order (reference graphs.py:251-276), so a given seed yields the same graph;
  * ``generate_erdos_renyi_gnm`` -- config 1's G(n, m), defined here;
  * ``generate_chung_lu`` -- config 4's power-law graph, defined here.
The last two are absent from the reference; their exact
definitions are documented in DESIGN.md.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

__all__ = ["CsrGraph", "DirectedView", "DeviceCsr", "degree_order",
           "generate_kronecker", "generate_erdos_renyi_gnm",
           "generate_chung_lu", "degree_stats", "DegreeStats"]


# ---------------------------------------------------------------------------
# device mirror


def _to_device(a, dtype):
    """Upload a host array (pinned memory is copied asynchronously) and cast
    on the device."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to("cuda", non_blocking=t.is_pinned()).to(dtype)


_SIDE_STREAMS = {}


def side_stream(name: str):
    """Process-wide auxiliary CUDA stream (copy / build overlap)."""
    import torch
    dev = torch.cuda.current_device()
    key = (name, dev)
    if key not in _SIDE_STREAMS:
        _SIDE_STREAMS[key] = torch.cuda.Stream()
    return _SIDE_STREAMS[key]


# pinned int32 adjacencies at least this large are uploaded in chunks
# (PG_UPLOAD_CHUNKS=0 disables the chunked path)
CHUNKED_UPLOAD_MIN_BYTES = 32 << 20
UPLOAD_CHUNKS = int(os.environ.get("PG_UPLOAD_CHUNKS", "8"))


class DeviceCsr:
    """Device copy of a CSR (graph or directed view) and derived edge lists.

    A pinned int32 adjacency of at least CHUNKED_UPLOAD_MIN_BYTES is uploaded
    on a copy stream in UPLOAD_CHUNKS vertex-range chunks with one event each
    (``upload_chunks``), so the first sketch build can start on a chunk as
    soon as it lands (sketches._build_on_device); the current stream waits for
    the whole upload, so every other consumer is ordered after it.
    """

    def __init__(self, offsets: np.ndarray, adjacency: np.ndarray):
        import torch
        if len(offsets) - 1 >= 2 ** 31:
            raise ValueError("vertex IDs must fit in int32 on the device")
        self.n = len(offsets) - 1
        self.nnz = len(adjacency)
        self.upload_chunks = []
        self.chunk_bounds = []  # (v0, v1, nnz_before) of every upload chunk
        adj_t = torch.from_numpy(np.ascontiguousarray(adjacency))
        if (UPLOAD_CHUNKS > 0 and adj_t.dtype == torch.int32 and adj_t.is_pinned()
                and adjacency.nbytes >= CHUNKED_UPLOAD_MIN_BYTES and self.n > 0):
            self._chunked_upload(np.asarray(offsets), adj_t)
        else:
            # host arrays go up as they are (int64 in the reference contract)
            # and are narrowed on the device: no host-side conversion pass
            self.offsets = _to_device(offsets, torch.int64)
            self.adj = _to_device(adjacency, torch.int32)
        self.degrees = (self.offsets[1:] - self.offsets[:-1]).to(torch.int32)
        self._upper = None
        self._src = None
        self._layouts = {}

    def _chunked_upload(self, offsets: np.ndarray, adj_t) -> None:
        import torch
        cur = torch.cuda.current_stream()
        cs = side_stream("copy")
        # the offsets go first (every chunk's build needs them), issued
        # before the rest of the setup: the copy engine is the critical path
        self.offsets = torch.empty(self.n + 1, dtype=torch.int64, device="cuda")
        off_t = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64))
        cs.wait_stream(cur)  # the new blocks may still be in use on cur
        with torch.cuda.stream(cs):
            self.offsets.copy_(off_t, non_blocking=True)
        self.adj = torch.empty(self.nnz, dtype=torch.int32, device="cuda")
        # equal-volume chunks (tapered tails and per-chunk offsets slices
        # measured slower: each extra DMA + build launch costs more than the
        # shorter tail saves).  int64 needles: float needles would convert
        # all of `offsets`.
        targets = (np.arange(UPLOAD_CHUNKS + 1, dtype=np.int64) * self.nnz) // UPLOAD_CHUNKS
        cuts = np.searchsorted(offsets, targets, side="left")
        cuts[0], cuts[-1] = 0, self.n
        cuts = np.unique(cuts)
        cs.wait_stream(cur)
        with torch.cuda.stream(cs):
            # highest vertex range first: once chunk c has landed, every
            # range above it is on the device, so a chunk's upper-triangle
            # edges (u < v) can be estimated as soon as its own sketches are
            # built (mining._tc_counts_chunked)
            for v0, v1 in reversed(list(zip(cuts[:-1].tolist(), cuts[1:].tolist()))):
                a, b = int(offsets[v0]), int(offsets[v1])
                if b > a:
                    self.adj[a:b].copy_(adj_t[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
                self.upload_chunks.append((v0, v1, ev))
                self.chunk_bounds.append((v0, v1, a, b))
        self.offsets.record_stream(cs)
        self.adj.record_stream(cs)
        cur.wait_stream(cs)

    def take_upload_chunks(self):
        """The pending (v0, v1, event) upload chunks, once (first consumer)."""
        chunks, self.upload_chunks = self.upload_chunks, []
        return chunks

    @classmethod
    def from_tensors(cls, offsets, adj) -> "DeviceCsr":
        """Wrap device tensors (int64 offsets, int32 adjacency) already in HBM."""
        import torch
        self = cls.__new__(cls)
        self.n = offsets.numel() - 1
        self.nnz = adj.numel()
        self.offsets = offsets
        self.adj = adj
        self.upload_chunks = []
        self.chunk_bounds = []
        self.degrees = (offsets[1:] - offsets[:-1]).to(torch.int32)
        self._upper = None
        self._src = None
        self._layouts = {}
        return self

    def upper_edges(self):
        """(us, vs) int32 device arrays: every undirected edge once, u < v."""
        if self._upper is None:
            import torch
            from . import _native as N
            m_alloc = max(1, self.nnz // 2)
            us = torch.empty(m_alloc, dtype=torch.int32, device="cuda")
            vs = torch.empty(m_alloc, dtype=torch.int32, device="cuda")
            import ctypes
            ws_bytes = ctypes.c_size_t()
            N.call("pg_csr_upper_edges_workspace", self.n, m_alloc, ctypes.byref(ws_bytes))
            ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8,
                             device="cuda")
            m = ctypes.c_int64()
            N.call("pg_csr_upper_edges", N.ptr(self.offsets), N.ptr(self.adj),
                   self.n, N.ptr(us), N.ptr(vs), m_alloc, ctypes.byref(m),
                   N.ptr(ws), ws_bytes.value, N.stream_handle())
            self._upper = (us[:m.value], vs[:m.value])
        return self._upper

    def upper_edges_padded(self, pad: int):
        """Row-padded upper edge slots (pad >= 2): (us, vs, slots), vs = -1 on
        padding slots; every aligned group of `pad` slots shares one u."""
        if pad <= 1:
            us, vs = self.upper_edges()
            return us, vs, us.numel()
        key = ("padded", pad)
        if key not in self._layouts:
            import ctypes
            import torch
            from . import _native as N
            # upper bound on slots: m + (pad-1) per non-empty row
            cap = self.nnz // 2 + (pad - 1) * self.n + 1
            us = torch.empty(cap, dtype=torch.int32, device="cuda")
            vs = torch.empty(cap, dtype=torch.int32, device="cuda")
            ws_bytes = ctypes.c_size_t()
            N.call("pg_csr_upper_edges_workspace", self.n, cap, ctypes.byref(ws_bytes))
            ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device="cuda")
            slots = ctypes.c_int64()
            N.call("pg_csr_upper_edges_padded", N.ptr(self.offsets), N.ptr(self.adj),
                   self.n, pad, N.ptr(us), N.ptr(vs), cap, ctypes.byref(slots),
                   N.ptr(ws), ws_bytes.value, N.stream_handle())
            k = slots.value
            self._layouts[key] = (us[:k], vs[:k], k)
        return self._layouts[key]

    def upper_edges_group_u(self, pad: int):
        """(ug, vs, slots) of the row-padded layout with one u per group of
        `pad` slots (ug[j // pad]), the group-u layout of pg_tc_bloom."""
        key = ("group_u", pad)
        if key not in self._layouts:
            us, vs, slots = self.upper_edges_padded(pad)
            self._layouts[key] = (us[::pad].contiguous(), vs, slots)
        return self._layouts[key]

    def degree_rank(self):
        """(rank int32[n], N+ offsets int64[n+1], N+ adjacency int32[m]):
        degree_order on the device (pg_degree_order), cached."""
        key = ("degree",)
        if key not in self._layouts:
            import torch
            from . import _native as N
            half = self.nnz // 2
            rank = torch.empty(max(1, self.n), dtype=torch.int32, device="cuda")
            off = torch.empty(self.n + 1, dtype=torch.int64, device="cuda")
            adj = torch.empty(max(1, half), dtype=torch.int32, device="cuda")
            N.call("pg_degree_order", N.ptr(self.offsets), N.ptr(self.adj), self.n, self.nnz,
                   N.ptr(rank), N.ptr(off), N.ptr(adj), N.stream_handle())
            self._layouts[key] = (rank[:self.n], off, adj[:half])
        return self._layouts[key]

    def hub_slots(self, pad: int, n_hubs: int):
        """Degree-oriented group-u slots with hub tags (pg_tc_bloom_hub):
        (ug, vs, slots, hub_ids).  Every edge once, from its lower- to its
        higher-(degree, ID)-rank endpoint (the N+ lists of degree_order),
        rows padded to `pad`; vs of the n_hubs highest-ranked vertices is
        the tag -2 - hub index, hub_ids maps it back."""
        key = ("hub", pad, n_hubs)
        if key not in self._layouts:
            import ctypes
            import torch
            from . import _native as N
            rank, off, adj = self.degree_rank()
            cap = adj.numel() + (pad - 1) * self.n + 1
            us = torch.empty(cap, dtype=torch.int32, device="cuda")
            vs = torch.empty(cap, dtype=torch.int32, device="cuda")
            ws_bytes = ctypes.c_size_t()
            N.call("pg_csr_upper_edges_workspace", self.n, cap, ctypes.byref(ws_bytes))
            ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device="cuda")
            slots = ctypes.c_int64()
            N.call("pg_csr_row_slots_padded", N.ptr(off), N.ptr(adj), self.n, pad, N.ptr(us),
                   N.ptr(vs), cap, ctypes.byref(slots), N.ptr(ws), ws_bytes.value,
                   N.stream_handle())
            k = slots.value
            hub_ids = torch.empty(max(1, n_hubs), dtype=torch.int32, device="cuda")
            N.call("pg_hub_tag", N.ptr(rank), self.n, n_hubs, N.ptr(vs), k, N.ptr(hub_ids),
                   N.stream_handle())
            del ws
            self._layouts[key] = (us[:k:pad].contiguous(), vs[:k], k, hub_ids)
        return self._layouts[key]

    def hybrid_slots(self, pad: int, thr: int, base: str = "degree"):
        """Degree-oriented group-u slots with less padding: (ug, vs, slots).
        The N+ rows keep their own slot groups (as hub_slots(pad, 0)) except
        for a last group of at most `thr` entries (the whole row when it has
        at most thr): those edges -- a few per cent of the edges, most of the
        pad slots at R-MAT -- are grouped by their higher-rank endpoint
        instead (its row is the one a group holds in registers), where they
        form long runs.  Every edge still appears once; which endpoint is
        called u only matters for the schedule.  base = "id" does the same
        over the upper-triangle lists (u < v by ID)."""
        key = ("hybrid", pad, thr, base)
        if key not in self._layouts:
            import ctypes
            import torch
            from . import _native as N
            n = self.n
            if base == "degree":
                _, off, adj = self.degree_rank()
            else:  # "id": the upper-triangle lists (u < v by ID)
                ts, adj = self.upper_edges()
                off = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
                off[1:] = torch.cumsum(torch.bincount(ts, minlength=n), 0)
            dplus = off[1:] - off[:-1]
            # a row's last (d+ mod pad) entries fill a slot group of their own:
            # when that remainder is at most thr they move to part 2 (for rows
            # of at most thr entries that is the whole row)
            rem = dplus % pad
            moved = torch.where((rem > 0) & (rem <= thr), rem, torch.zeros_like(rem))
            kept = dplus - moved
            src = torch.repeat_interleave(torch.arange(n, dtype=torch.int32, device="cuda"), dplus)
            pos = torch.arange(adj.numel(), dtype=torch.int64, device="cuda") - off[:-1][src.long()]
            keep = pos < kept[src.long()]
            del pos
            # part 1: the kept entries by their own (lower-rank) vertex
            off1 = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
            off1[1:] = torch.cumsum(kept, 0)
            adj1 = adj[keep].contiguous()
            # part 2: the short rows' edges by the higher-rank endpoint
            lo, hi = src[~keep], adj[~keep]
            del src, keep
            order = torch.sort(hi.long(), stable=True).indices
            adj2 = lo[order].contiguous()
            off2 = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
            off2[1:] = torch.cumsum(torch.bincount(hi, minlength=n), 0)
            del lo, hi, order
            parts = []
            for o, a in ((off1, adj1), (off2, adj2)):
                cap = a.numel() + (pad - 1) * n + 1
                us = torch.empty(cap, dtype=torch.int32, device="cuda")
                vs = torch.empty(cap, dtype=torch.int32, device="cuda")
                ws_bytes = ctypes.c_size_t()
                N.call("pg_csr_upper_edges_workspace", n, cap, ctypes.byref(ws_bytes))
                ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device="cuda")
                slots = ctypes.c_int64()
                N.call("pg_csr_row_slots_padded", N.ptr(o), N.ptr(a), n, pad, N.ptr(us), N.ptr(vs), cap,
                       ctypes.byref(slots), N.ptr(ws), ws_bytes.value, N.stream_handle())
                k = slots.value
                parts.append((us[:k:pad], vs[:k], k))
                del ws
            # the two parts interleaved in 64 segments each, so that any
            # contiguous share of the slots (a rank's shard) holds the same mix
            # (part 2 streams low-degree rows from HBM and runs ~13 % slower
            # per slot: with it at the end the last of 8 shards took 0.644 ms
            # against 0.57 for the others)
            seg = 64
            ugs, vss = [], []
            for i in range(seg):
                for g_arr, v_arr, k in parts:
                    groups = k // pad
                    a, b = groups * i // seg, groups * (i + 1) // seg
                    ugs.append(g_arr[a:b])
                    vss.append(v_arr[a * pad:b * pad])
            ug = torch.cat(ugs)
            vs = torch.cat(vss)
            self._layouts[key] = (ug, vs, parts[0][2] + parts[1][2])
        return self._layouts[key]

    def max_degree(self) -> int:
        """Largest row length (one device reduction, cached)."""
        if getattr(self, "_maxd", None) is None:
            self._maxd = int(self.degrees.max().item()) if self.n > 0 else 0
        return self._maxd

    def row_sources(self):
        """int32 device array src[j] = row of adjacency entry j."""
        if self._src is None:
            import torch
            from . import _native as N
            src = torch.empty(max(1, self.nnz), dtype=torch.int32, device="cuda")
            N.call("pg_csr_expand_rows", N.ptr(self.offsets), self.n, self.nnz,
                   N.ptr(src), N.stream_handle())
            self._src = src[:self.nnz]
        return self._src


# ---------------------------------------------------------------------------
# host CSR


class CsrGraph:
    """Undirected simple graph in CSR form (reference graphs.py:32-129)."""

    __slots__ = ("n", "m", "offsets", "adjacency", "original_ids",
                 "self_loops_dropped", "duplicates_dropped", "_dev")

    def __init__(self, offsets, adjacency, original_ids=None):
        self.offsets = np.asarray(offsets, dtype=np.int64)
        adjacency = np.asarray(adjacency)
        # int64 as in the reference; an int32 adjacency (BASELINE's "int32
        # CSR") is kept as is, halving the host->device copy
        if adjacency.dtype != np.int32:
            adjacency = adjacency.astype(np.int64, copy=False)
        self.adjacency = adjacency
        self.n = len(self.offsets) - 1
        self.m = len(self.adjacency) // 2
        self.original_ids = original_ids
        self.self_loops_dropped = 0
        self.duplicates_dropped = 0
        self._dev = None

    @classmethod
    def from_edges(cls, edges, n: int | None = None) -> "CsrGraph":
        """Symmetrise, deduplicate and drop self loops (reference
        graphs.py:57-89).  On a CUDA machine the pairs are canonicalised,
        sorted and deduplicated on the device (pg_csr_from_pairs) and the
        graph keeps its device mirror."""
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        if len(e) and int(e.min()) < 0:
            raise ValueError("vertex IDs must be non-negative")
        if len(e) and _cuda_available():
            return cls._from_edges_device(e, n)
        lo = np.minimum(e[:, 0], e[:, 1])
        hi = np.maximum(e[:, 0], e[:, 1])
        proper = lo != hi
        loops = int(len(e) - np.count_nonzero(proper))
        lo, hi = lo[proper], hi[proper]
        if n is None:
            n = int(hi.max()) + 1 if len(hi) else 0
        if len(hi) and int(hi.max()) >= n:
            raise ValueError("edge endpoint exceeds vertex count")
        # canonical pair key; n < 2**31 keeps n*n inside int64
        key = np.unique(lo * n + hi)
        dups = len(lo) - len(key)
        g = cls._from_canonical_keys(key, n)
        g.self_loops_dropped = loops
        g.duplicates_dropped = int(dups)
        return g

    @classmethod
    def _from_edges_device(cls, e: np.ndarray, n: int | None) -> "CsrGraph":
        import torch
        t = torch.from_numpy(np.ascontiguousarray(e)).cuda()
        a, b = t[:, 0].contiguous(), t[:, 1].contiguous()
        proper = a != b
        loops = int(e.shape[0] - int(proper.sum().item()))
        hi_max = int(torch.where(proper, torch.maximum(a, b),
                                 torch.full_like(a, -1)).max().item())
        if n is None:
            n = hi_max + 1 if hi_max >= 0 else 0
        if hi_max >= n:
            raise ValueError("edge endpoint exceeds vertex count")
        if n >= 2 ** 31:
            raise ValueError("vertex IDs must fit in int32 on the device")
        if loops == e.shape[0]:  # nothing but self loops: the empty graph
            g = cls._from_canonical_keys(np.empty(0, dtype=np.int64), n)
        else:
            g = _graph_from_device_pairs(a, b, n)
            g.adjacency = g.adjacency.astype(np.int64)  # the reference's dtype
        g.self_loops_dropped = loops
        g.duplicates_dropped = int(e.shape[0] - loops - g.m)
        return g

    @classmethod
    def _from_canonical_keys(cls, key: np.ndarray, n: int) -> "CsrGraph":
        """CSR from sorted unique keys lo*n+hi (lo < hi)."""
        if n == 0:
            return cls(np.zeros(1, dtype=np.int64), np.empty(0, dtype=np.int64))
        lo, hi = np.divmod(key, n)
        both = np.concatenate([lo * n + hi, hi * n + lo])
        del lo, hi
        both.sort(kind="stable")
        src, dst = np.divmod(both, n)
        del both
        counts = np.bincount(src, minlength=n)
        offsets = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=offsets[1:])
        return cls(offsets, dst)

    def neighbors(self, v: int) -> np.ndarray:
        return self.adjacency[self.offsets[v]:self.offsets[v + 1]]

    def degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])

    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets)

    def edges(self) -> np.ndarray:
        """(m, 2) int64: each undirected edge once, u < v, CSR order."""
        src = np.repeat(np.arange(self.n, dtype=np.int64), self.degrees())
        upper = src < self.adjacency
        return np.stack([src[upper], self.adjacency[upper]], axis=1)

    def validate(self) -> None:
        if len(self.offsets) != self.n + 1 or (self.n >= 0 and self.offsets[0] != 0):
            raise ValueError("bad offsets")
        if np.any(np.diff(self.offsets) < 0):
            raise ValueError("offsets not non-decreasing")
        if self.offsets[-1] != len(self.adjacency) or len(self.adjacency) % 2:
            raise ValueError("offsets[n] != 2m")
        src = np.repeat(np.arange(self.n, dtype=np.int64), self.degrees())
        key = src * max(self.n, 1) + self.adjacency
        if len(key) and np.any(np.diff(key) <= 0):
            raise ValueError("neighbourhoods not sorted/unique")
        if np.any(src == self.adjacency):
            raise ValueError("self loop")
        rev = np.sort(self.adjacency * max(self.n, 1) + src)
        if not np.array_equal(rev, key):
            raise ValueError("adjacency not symmetric")

    def device(self) -> DeviceCsr:
        """Device mirror (built on first use, then cached)."""
        if self._dev is None:
            self._dev = DeviceCsr(self.offsets, self.adjacency)
        return self._dev


@dataclass(frozen=True)
class DirectedView:
    """Degree-ordered orientation (reference graphs.py:132-166)."""

    n: int
    m: int
    rank: np.ndarray
    offsets: np.ndarray
    adjacency: np.ndarray
    _dev: list = field(default_factory=list, repr=False, compare=False)

    def out_neighbors(self, v: int) -> np.ndarray:
        return self.adjacency[self.offsets[v]:self.offsets[v + 1]]

    def out_degrees(self) -> np.ndarray:
        return np.diff(self.offsets)

    def device(self) -> DeviceCsr:
        if not self._dev:
            self._dev.append(DeviceCsr(self.offsets, self.adjacency))
        return self._dev[0]


def as_csr_graph(graph) -> CsrGraph:
    """This package's CsrGraph for any object with the reference CsrGraph's
    ``offsets`` / ``adjacency`` arrays (graphs.py:32-56) -- e.g. a graph
    built by the reference itself.  The wrapper is cached on the object, so
    its device mirror is uploaded once."""
    if isinstance(graph, CsrGraph):
        return graph
    try:
        offsets, adjacency = graph.offsets, graph.adjacency
    except AttributeError as exc:
        raise TypeError(f"expected a CSR graph (offsets, adjacency): {exc}") from None
    cached = _ADOPTED.get(id(graph))
    if cached is not None and cached[0] is graph:
        return cached[1]
    g = CsrGraph(offsets, adjacency, getattr(graph, "original_ids", None))
    _ADOPTED[id(graph)] = (graph, g)
    return g


def as_directed_view(view) -> DirectedView:
    """This package's DirectedView for any object with the reference
    DirectedView fields (n, m, rank, offsets, adjacency; graphs.py:132-151)."""
    if isinstance(view, DirectedView):
        return view
    try:
        fields = (int(view.n), int(view.m), np.asarray(view.rank, dtype=np.int64),
                  np.asarray(view.offsets, dtype=np.int64), np.asarray(view.adjacency))
    except AttributeError as exc:
        raise TypeError(f"expected a degree-ordered view: {exc}") from None
    cached = _ADOPTED.get(id(view))
    if cached is not None and cached[0] is view:
        return cached[1]
    v = DirectedView(*fields)
    _ADOPTED[id(view)] = (view, v)
    return v


# id(foreign object) -> (object, adopted wrapper); keeps the object alive so
# the id is not reused while the entry exists
_ADOPTED: dict = {}


def degree_order(graph: CsrGraph) -> DirectedView:
    """Keep u in N+(v) iff (deg v, v) < (deg u, u) (reference graphs.py:154-166).

    On a CUDA machine the ranking and the directed CSR are built on the
    device (pg_degree_order) and the view keeps them resident; host arrays
    are copied back for the reference contract.
    """
    graph = as_csr_graph(graph)
    if graph.n > 0 and _cuda_available():
        return _degree_order_device(graph)
    return _degree_order_host(graph)


def _degree_order_device(graph: CsrGraph) -> DirectedView:
    import torch
    from . import _native as N
    dev = graph.device()
    half = dev.nnz // 2
    rank = torch.empty(graph.n, dtype=torch.int32, device="cuda")
    off = torch.empty(graph.n + 1, dtype=torch.int64, device="cuda")
    adj = torch.empty(max(1, half), dtype=torch.int32, device="cuda")
    N.call("pg_degree_order", N.ptr(dev.offsets), N.ptr(dev.adj), graph.n, dev.nnz,
           N.ptr(rank), N.ptr(off), N.ptr(adj), N.stream_handle())
    adj = adj[:half]
    host_adj = adj.cpu().numpy()
    if graph.adjacency.dtype != np.int32:
        host_adj = host_adj.astype(np.int64)
    view = DirectedView(graph.n, graph.m, rank.cpu().numpy().astype(np.int64),
                        off.cpu().numpy(), host_adj)
    view._dev.append(DeviceCsr.from_tensors(off, adj))
    return view


def _degree_order_host(graph: CsrGraph) -> DirectedView:
    deg = graph.degrees()
    order = np.argsort(deg, kind="stable")  # ties -> ascending ID
    rank = np.empty(graph.n, dtype=np.int64)
    rank[order] = np.arange(graph.n, dtype=np.int64)
    src = np.repeat(np.arange(graph.n, dtype=np.int64), deg)
    keep = rank[src] < rank[graph.adjacency]
    out_src = src[keep]
    counts = np.bincount(out_src, minlength=graph.n)
    offsets = np.zeros(graph.n + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return DirectedView(graph.n, graph.m, rank, offsets, graph.adjacency[keep])


# ---------------------------------------------------------------------------
# generators


def _cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def _pcg64_state(rng) -> tuple[int, int, int, int]:
    """(state_hi, state_lo, inc_hi, inc_lo) of numpy's PCG64 bit generator."""
    st = rng.bit_generator.state["state"]
    m64 = (1 << 64) - 1
    return (st["state"] >> 64, st["state"] & m64, st["inc"] >> 64, st["inc"] & m64)


def _graph_from_device_pairs(a, b, n: int) -> CsrGraph:
    """CsrGraph.from_edges on the device (pg_csr_from_pairs); the returned
    graph carries its device mirror, host arrays are copied back once."""
    import ctypes
    import torch
    from . import _native as N
    off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    adj = torch.empty(max(1, 2 * a.numel()), dtype=torch.int32, device="cuda")
    nnz = ctypes.c_int64()
    N.call("pg_csr_from_pairs", N.ptr(a), N.ptr(b), a.numel(), n, N.ptr(off),
           N.ptr(adj), adj.numel(), ctypes.byref(nnz), N.stream_handle())
    adj = adj[:nnz.value].clone()
    g = CsrGraph(off.cpu().numpy(), adj.cpu().numpy())
    g._dev = DeviceCsr.from_tensors(off, adj)
    return g


def generate_kronecker(scale: int, edge_factor: int, seed: int,
                       device: bool | None = None) -> CsrGraph:
    """R-MAT, initiator (a, b, c, d) = (0.57, 0.19, 0.19, 0.05).

    Per level l (LSB first) each sample draws ``rng.random(count)`` for the
    source bit, then ``rng.random(count)`` for the destination bit whose
    threshold depends on the source bit -- the reference's draw order, so
    graphs are identical for a given seed.  With a CUDA device (default when
    one is present) the same PCG64 stream is generated on the device
    (pg_rmat_pairs) and deduplicated there (pg_csr_from_pairs).
    """
    if scale < 1:
        raise ValueError("scale must be >= 1")
    n = 1 << scale
    count = edge_factor * n
    rng = np.random.default_rng(seed)
    if device is None:
        device = _cuda_available()
    if device:
        import torch
        from . import _native as N
        src = torch.empty(max(1, count), dtype=torch.int64, device="cuda")
        dst = torch.empty(max(1, count), dtype=torch.int64, device="cuda")
        N.call("pg_rmat_pairs", *_pcg64_state(rng), scale, count, 0.57, 0.19,
               0.19, N.ptr(src), N.ptr(dst), N.stream_handle())
        return _graph_from_device_pairs(src[:count], dst[:count], n)
    p_ab = 0.57 + 0.19
    thr_given_src0 = 0.57 / p_ab            # P(dst bit 0 | src bit 0)
    thr_given_src1 = 0.19 / (1.0 - p_ab)    # P(dst bit 0 | src bit 1)
    src = np.zeros(count, dtype=np.int64)
    dst = np.zeros(count, dtype=np.int64)
    thr = np.empty(count, dtype=np.float64)
    for level in range(scale):
        sbit = rng.random(count) > p_ab
        np.copyto(thr, thr_given_src0)
        thr[sbit] = thr_given_src1
        dbit = rng.random(count) > thr
        src |= sbit.astype(np.int64) << level
        dst |= dbit.astype(np.int64) << level
    del thr
    return CsrGraph.from_edges(np.stack([src, dst], axis=1), n=n)


def generate_erdos_renyi_gnm(n: int, m: int, seed: int) -> CsrGraph:
    """Uniform simple graph with exactly m edges (config 1).

    Draws batches of endpoint pairs ``rng.integers(0, n, size=(B, 2))``,
    drops self loops, and keeps each unordered pair at its first occurrence
    in draw order until m distinct pairs are collected.
    """
    if m > n * (n - 1) // 2:
        raise ValueError("too many edges for a simple graph")
    rng = np.random.default_rng(seed)
    chosen = np.empty(0, dtype=np.int64)
    while len(chosen) < m:
        batch = int((m - len(chosen)) * 1.25) + 1024
        pairs = rng.integers(0, n, size=(batch, 2), dtype=np.int64)
        lo = np.minimum(pairs[:, 0], pairs[:, 1])
        hi = np.maximum(pairs[:, 0], pairs[:, 1])
        key = (lo * n + hi)[lo != hi]
        uniq, first = np.unique(key, return_index=True)
        fresh = ~np.isin(uniq, chosen)
        new_keys = key[np.sort(first[fresh])]
        chosen = np.concatenate([chosen, new_keys[:m - len(chosen)]])
    return CsrGraph._from_canonical_keys(np.sort(chosen), n)


def generate_chung_lu(n: int, avg_degree: float, gamma: float, seed: int,
                      weight_cap: float | None = None,
                      device: bool | None = None) -> CsrGraph:
    """Chung-Lu power-law graph (config 4).

    Weights w_i = (i+1)^(-1/(gamma-1)) scaled to mean ``avg_degree`` and capped
    at ``weight_cap`` (default sqrt(n * avg_degree), the structural cutoff),
    then M = round(n * avg_degree / 2) edge samples draw both endpoints
    independently with probability proportional to w (inverse-CDF on
    ``rng.random(M)`` for u, then for v); the result is symmetrised,
    deduplicated and loop-free.  Vertex 0 carries the largest weight.
    """
    if gamma <= 2.0:
        raise ValueError("gamma must exceed 2")
    rng = np.random.default_rng(seed)
    w = np.arange(1, n + 1, dtype=np.float64) ** (-1.0 / (gamma - 1.0))
    w *= avg_degree * n / w.sum()
    cap = float(np.sqrt(n * avg_degree)) if weight_cap is None else weight_cap
    np.minimum(w, cap, out=w)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    samples = int(round(n * avg_degree / 2.0))
    if device is None:
        device = _cuda_available()
    if device:
        import torch
        from . import _native as N
        st = _pcg64_state(rng)
        cdf_d = torch.from_numpy(cdf).cuda()
        draws = torch.empty(max(1, samples), dtype=torch.float64, device="cuda")
        ends = []
        for offset in (0, samples):  # u from the first rng.random, v the second
            N.call("pg_pcg64_uniform", *st, offset, samples, N.ptr(draws),
                   N.stream_handle())
            out = torch.empty(max(1, samples), dtype=torch.int64, device="cuda")
            N.call("pg_searchsorted_right", N.ptr(cdf_d), n, N.ptr(draws), samples,
                   N.ptr(out), N.stream_handle())
            ends.append(out[:samples])
        return _graph_from_device_pairs(ends[0], ends[1], n)
    u = np.searchsorted(cdf, rng.random(samples), side="right")
    v = np.searchsorted(cdf, rng.random(samples), side="right")
    np.minimum(u, n - 1, out=u)
    np.minimum(v, n - 1, out=v)
    return CsrGraph.from_edges(np.stack([u, v], axis=1), n=n)


@dataclass(frozen=True)
class DegreeStats:
    max_degree: int
    mean_degree: float
    sum_d2: int
    sum_d3: int


def degree_stats(graph: CsrGraph) -> DegreeStats:
    d = graph.degrees().astype(np.int64)
    if graph.n == 0:
        return DegreeStats(0, 0.0, 0, 0)
    return DegreeStats(int(d.max(initial=0)), float(d.mean()),
                       int((d * d).sum()), int((d * d * d).sum()))
