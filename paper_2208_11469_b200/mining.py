"""Mining entry points on the device (the callers of the per-edge path).

Same names and signatures as reference ``mining.py``: ``triangle_count``
(:88-102), ``tc_estimate`` (:105-130), ``four_clique_count`` (:133-154),
``vertex_similarity`` (:162-203), ``jarvis_patrick_cluster`` (:213-245).
``threads`` is accepted for compatibility; the device does the fan-out.

Where the reference sums per-edge floats over a fixed 16,384-edge chunk grid
(:63-80), the device kernels reduce exact integer statistics (popcount
histograms, per-match-count sums) that the host turns into the estimate with
``math.fsum``; the result agrees with the reference to ~1e-15 relative and is
independent of the grid, the shard count and the thread count.

``jaccard_cluster_count`` is the config-4 entry point (k-Hash Jaccard >= tau,
count surviving edges); the reference has no batch form of it.
"""

from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .estimators import EstimatorKind, swamidass_table
from .graphs import CsrGraph, DirectedView, as_csr_graph, as_directed_view, degree_order
from .providers import (BloomProvider, ExactProvider, IntersectionProvider, KmvProvider,
                        MinHashProvider, UnsupportedCombinationError, make_provider)
from .sketches import SketchedGraph, SketchKind, as_sketched_graph

__all__ = ["SimilarityMeasure", "ClusterResult", "JaccardCount", "LinkPredSplit",
           "triangle_count", "tc_estimate", "tc_counts", "four_clique_count",
           "vertex_similarity", "jarvis_patrick_cluster",
           "jaccard_cluster_count", "jaccard_min_matches",
           "make_link_prediction_split", "link_prediction_eval",
           "doulion_tc", "reduced_execution_tc"]


class SimilarityMeasure(str, enum.Enum):
    JACCARD = "jaccard"
    OVERLAP = "overlap"
    COMMON_NEIGHBORS = "common_neighbors"
    TOTAL_NEIGHBORS = "total_neighbors"
    ADAMIC_ADAR = "adamic_adar"
    RESOURCE_ALLOCATION = "resource_allocation"


_COUNTING = (SimilarityMeasure.JACCARD, SimilarityMeasure.OVERLAP,
             SimilarityMeasure.COMMON_NEIGHBORS, SimilarityMeasure.TOTAL_NEIGHBORS)


def _is_exact(kind: EstimatorKind) -> bool:
    return kind in (EstimatorKind.EXACT_MERGE, EstimatorKind.EXACT_GALLOP)


def triangle_count(view: DirectedView, provider: IntersectionProvider,
                   threads: int = 1):
    """Sum of |N+v & N+u| over directed edges (exact int for exact providers)."""
    view = as_directed_view(view)
    dev = view.device()
    if isinstance(provider, ExactProvider):
        # fused intersections + sum over the provider's CSR
        import torch
        d = provider.device()
        out = torch.empty(1, dtype=torch.int64, device="cuda")
        N.call("pg_tc_exact", N.ptr(d.offsets), N.ptr(d.adj), N.ptr(dev.row_sources()),
               N.ptr(dev.adj), dev.nnz, N.ptr(out), N.stream_handle())
        return int(out.item())
    part = provider._pairs_device(dev.row_sources(), dev.adj)
    if provider.is_exact:
        return int(part.sum().item()) if part.numel() else 0
    return float(part.sum().item()) if part.numel() else 0.0


def _tc_provider(graph: CsrGraph, sketched, kind):
    kind = EstimatorKind(getattr(kind, "value", kind))
    if sketched is not None:
        sketched = as_sketched_graph(sketched)
    if _is_exact(kind):
        return make_provider(kind, graph=graph)
    if sketched is None:
        raise ValueError("sketch-based estimate needs a SketchedGraph")
    if sketched.source != "undirected":
        raise ValueError("triangle-count estimation needs sketches of the "
                         "undirected neighborhoods")
    return make_provider(kind, sketched=sketched)


def tc_counts(provider, dev, rank: int = 0, world: int = 1):
    """Device partial statistics of this rank's share of the edge slots:
    int64 histograms / per-match sums (fp64 sum for KMV), see _tc_combine."""
    import torch
    from .sharding import edge_range
    if provider.is_exact:
        us, vs = dev.upper_edges()
        b, e = edge_range(us.numel(), rank, world)
        part = provider._pairs_device(us[b:e], vs[b:e])
        return part.sum().reshape(1) if part.numel() else torch.zeros(
            1, dtype=torch.int64, device="cuda")
    if world == 1 and _chunk_pipelined(provider, dev):
        return _tc_counts_chunked(provider, dev)
    lay = provider._tc_layout(dev)
    return provider._tc_counts_shard(lay, rank, world)


def _chunk_pipelined(provider, dev) -> bool:
    """A Bloom TC whose CSR is still arriving in upload chunks with per-chunk
    sketch builds (the host-CSR path): it can run chunk by chunk."""
    sg = getattr(provider, "sketched", None)
    return (isinstance(provider, BloomProvider) and provider.kind is not EstimatorKind.BF_OR
            and sg is not None and bool(sg._chunk_ready) and sg._chunk_dev is dev
            and provider.tc_pad() > 1 and not dev._layouts)


def _tc_counts_chunked(provider, dev):
    """The fused Bloom TC of a chunk-uploaded graph, pipelined with the
    upload.  Chunks arrive highest vertex range first (DeviceCsr), so the
    upper-triangle slots of chunk c (rows [v0, v1), neighbours > u, whose
    sketches are all built once c's are) are laid out on a side stream as
    soon as the chunk lands, and its TC runs on another as soon as its
    sketches are built, with device-side slot ranges (no host sync).  The
    slots are the whole-graph layout's, range by range: the same per-edge
    popcounts, so the same histogram."""
    import ctypes
    import torch
    from .graphs import side_stream
    sg = provider.sketched
    # the raw device buffers: device_tensors() would order the current
    # stream after the whole build; here each chunk waits for its own events
    d = sg._dev
    pad = provider.tc_pad()
    bits = sg.bit_length
    cur = torch.cuda.current_stream()
    ls, ts = side_stream("layout"), side_stream("tc")
    chunks = sg._chunk_ready
    cap = dev.nnz + (pad - 1) * dev.n + pad  # upper entries <= nnz: never overflows
    nnz_of = {(v0, v1): b - a for v0, v1, a, b in dev.chunk_bounds}

    def bound(v0, v1):  # host bound on a range's padded slots
        return nnz_of.get((v0, v1), dev.nnz) + (pad - 1) * (v1 - v0)

    max_rows = max(v1 - v0 for v0, v1, _, _ in chunks)
    ws_bytes = ctypes.c_size_t()
    N.call("pg_csr_range_slots_workspace", max_rows,
           max(bound(v0, v1) for v0, v1, _, _ in chunks), ctypes.byref(ws_bytes))
    with torch.cuda.stream(ls):
        ug = torch.empty(cap // pad + 1, dtype=torch.int32, device="cuda")
        vs = torch.empty(cap, dtype=torch.int32, device="cuda")
        ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device="cuda")
        cur_rng = torch.zeros(2 + 2 * len(chunks), dtype=torch.int64, device="cuda")
    with torch.cuda.stream(ts):
        out = torch.zeros(bits + 2, dtype=torch.int64, device="cuda")
    hl, h = N.stream_handle(ls), N.stream_handle(ts)
    for c, (v0, v1, copied, built) in enumerate(chunks):
        ls.wait_event(copied)
        rng = N.ptr(cur_rng) + 8 * (2 + 2 * c)
        max_slots = bound(v0, v1)
        N.call("pg_csr_range_slots_append", N.ptr(dev.offsets), N.ptr(dev.adj), v0, v1,
               pad, 0, max_slots, N.ptr(ug), N.ptr(vs), cap, N.ptr(cur_rng), rng,
               N.ptr(ws), ws_bytes.value, hl)
        laid = torch.cuda.Event()
        laid.record(ls)
        ts.wait_event(laid)
        ts.wait_event(built)
        # AND / L histograms need neither sizes nor the table (BF_OR does;
        # it takes the whole-graph path)
        N.call("pg_tc_bloom_range", N.ptr(d["rows"]), bits, provider.op,
               None, None, N.ptr(ug), N.ptr(vs), rng, max_slots, 1,
               N.ptr(out), N.ptr(out) + 8 * (bits + 1), h)
    for t in (ug, vs, cur_rng):  # read on ts after their last use on ls
        t.record_stream(ts)
    cur.wait_stream(ts)
    out.record_stream(cur)
    # cur_rng[1]: a range's slots exceeded its bound (they were dropped); the
    # bounds above cannot be exceeded, so this is an internal error
    if int(cur_rng[1].item()) != 0:
        raise N.EngineError("edge-slot range overflow in the chunked TC layout")
    return out


def tc_combine(provider, counts: np.ndarray) -> float:
    """Sum over edges of the per-edge estimates, from tc_counts outputs."""
    if provider.is_exact:
        return float(int(counts[0]))
    return provider._tc_combine(counts)


def tc_estimate(graph: CsrGraph, sketched: SketchedGraph | None = None,
                kind=EstimatorKind.BF_AND, threads: int = 1) -> float:
    """(1/3) * sum over undirected edges of the intersection estimate."""
    graph = as_csr_graph(graph)
    provider = _tc_provider(graph, sketched, kind)
    counts = tc_counts(provider, graph.device()).cpu().numpy()
    return tc_combine(provider, counts) / 3.0


def four_clique_count(view: DirectedView, provider: IntersectionProvider,
                      threads: int = 1):
    """sum over directed (u,v), w in C3 = N+u & N+v of |S_w & C3|
    (reference mining.py:133-154).

    Exact providers give the exact integer count, with N(w) from the
    provider's own CSR (``ExactProvider._slice``); Bloom providers estimate
    |N+w & C3| from BF+(w) and BF(C3) (fused kernel, integer histogram);
    k-Hash / 1-Hash / KMV providers build the member sketch of C3 once per
    directed edge on the device and add ``with_set``'s estimate for every w
    in C3 (pg_4clique_sketch).
    """
    import torch
    view = as_directed_view(view)
    dev = view.device()
    src, nnz = dev.row_sources(), dev.nnz
    if isinstance(provider, ExactProvider):
        pdev = provider.device()
        if pdev.n < view.n:
            raise ValueError("exact provider covers fewer vertices than the view")
        out = torch.empty(1, dtype=torch.int64, device="cuda")
        N.call("pg_4clique_exact_rows", N.ptr(dev.offsets), N.ptr(dev.adj), N.ptr(src),
               0, nnz, N.ptr(pdev.offsets), N.ptr(pdev.adj), N.ptr(out), N.stream_handle())
        return int(out.item())
    if isinstance(provider, BloomProvider):
        counts = four_clique_counts(view, provider, 0, nnz).cpu().numpy()
        return four_clique_combine(provider, counts)
    if isinstance(provider, (MinHashProvider, KmvProvider)):
        total, _ = four_clique_sketch_sum(view, provider)
        return total
    raise UnsupportedCombinationError(
        f"four_clique_count on the device supports exact, Bloom, MinHash and KMV "
        f"providers, not {type(provider).__name__}")


_C4_KIND = {SketchKind.KHASH: 3, SketchKind.ONEHASH: 4, SketchKind.KMV: 5}


def four_clique_sketch_sum(view: DirectedView, provider, edge_ids=None):
    """(sum of with_set estimates, triple count) over every directed edge of
    the view, or over the directed-edge indices ``edge_ids`` (a sample), for
    a k-Hash / 1-Hash / KMV provider (pg_4clique_sketch)."""
    import torch
    view = as_directed_view(view)
    dev = view.device()
    sg = provider.sketched
    if sg.n < view.n:
        raise ValueError("sketches cover fewer vertices than the view")
    d = sg.device_tensors()
    kind = _C4_KIND[sg.kind]
    k = sg.capacity
    maxd = dev.max_degree()
    ws_bytes = ctypes.c_size_t(0)
    N.call("pg_4clique_sketch_workspace_size", kind, k, maxd, ctypes.byref(ws_bytes))
    ws = torch.empty(max(16, ws_bytes.value), dtype=torch.uint8, device="cuda")
    out_sum = torch.empty(1, dtype=torch.float64, device="cuda")
    out_trip = torch.empty(1, dtype=torch.int64, device="cuda")
    rows = d["values"] if sg.kind is SketchKind.KMV else d["entries"]
    lengths = d.get("lengths") if sg.kind is not SketchKind.KHASH else None
    if edge_ids is None:
        ids, e0, e1 = None, 0, dev.nnz
    else:
        ids = torch.as_tensor(np.asarray(edge_ids, dtype=np.int64)
                              if not isinstance(edge_ids, torch.Tensor) else edge_ids)
        ids = ids.to(device="cuda", dtype=torch.int64).contiguous()
        if ids.numel() and (int(ids.min()) < 0 or int(ids.max()) >= dev.nnz):
            raise ValueError("edge id out of range")
        e0, e1 = 0, ids.numel()
    N.call("pg_4clique_sketch", kind, N.ptr(dev.offsets), N.ptr(dev.adj),
           N.ptr(dev.row_sources()), N.ptr(ids) if ids is not None else None, e0, e1,
           N.ptr(rows), N.ptr(lengths) if lengths is not None else None, N.ptr(d["sizes"]),
           k, N.ptr(d["seeds"]), maxd, N.ptr(ws), ws.numel(), N.ptr(out_sum),
           N.ptr(out_trip), N.stream_handle())
    return float(out_sum.item()), int(out_trip.item())


def four_clique_counts(view: DirectedView, provider: BloomProvider,
                       e_begin: int, e_end: int, edge_ids=None):
    """Device int64 [hist(B+1), sum_pos, triples] for the directed edges
    [e_begin, e_end), or for the directed-edge indices `edge_ids` (a sample;
    host or device int64) when given."""
    import torch
    dev = view.device()
    sg = provider.sketched
    d = sg.device_tensors()
    bits = sg.bit_length
    hist = torch.empty(bits + 1, dtype=torch.int64, device="cuda")
    spos = torch.empty(1, dtype=torch.int64, device="cuda")
    trip = torch.empty(1, dtype=torch.int64, device="cuda")
    tail = (N.ptr(d["rows"]), bits, sg.hash_count, N.ptr(d["seeds"]), provider.op,
            N.ptr(d["sizes"]), N.ptr(provider.lut_device()), N.ptr(hist), N.ptr(spos),
            N.ptr(trip), N.stream_handle())
    if edge_ids is None:
        N.call("pg_4clique_bloom", N.ptr(dev.offsets), N.ptr(dev.adj),
               N.ptr(dev.row_sources()), e_begin, e_end, *tail)
    else:
        ids = torch.as_tensor(np.asarray(edge_ids, dtype=np.int64)
                              if not isinstance(edge_ids, torch.Tensor) else edge_ids)
        ids = ids.to(device="cuda", dtype=torch.int64).contiguous()
        if ids.numel() and (int(ids.min()) < 0 or int(ids.max()) >= dev.nnz):
            raise ValueError("edge id out of range")
        N.call("pg_4clique_bloom_edges", N.ptr(dev.offsets), N.ptr(dev.adj),
               N.ptr(dev.row_sources()), N.ptr(ids), ids.numel(), *tail)
    return torch.cat([hist, spos, trip])


def four_clique_combine(provider: BloomProvider, counts: np.ndarray) -> float:
    return provider._tc_combine(counts[:-1])


def _feasible(c: float, du: int, dv: int) -> float:
    return min(max(c, 0.0), float(min(du, dv)))


def vertex_similarity(u: int, v: int, measure, provider: IntersectionProvider,
                      graph: CsrGraph) -> float:
    if u == v:
        raise ValueError("vertex similarity needs two distinct vertices")
    graph = as_csr_graph(graph)
    measure = SimilarityMeasure(getattr(measure, "value", measure))
    du, dv = graph.degree(u), graph.degree(v)
    if measure in _COUNTING:
        c = float(provider.pair(u, v))
        if measure is SimilarityMeasure.COMMON_NEIGHBORS:
            return c
        c = _feasible(c, du, dv)
        if measure is SimilarityMeasure.JACCARD:
            denom = du + dv - c
            return c / denom if denom > 0 else 0.0
        if measure is SimilarityMeasure.OVERLAP:
            lo = min(du, dv)
            return c / lo if lo > 0 else 0.0
        return du + dv - c
    members = provider.common_members(u, v)
    degs = graph.degrees()[members] if len(members) else np.empty(0)
    # sequential sums in member (ascending ID) order, as the reference
    # (mining.py:192-203) -- not fsum, whose rounding differs
    total = 0.0
    if measure is SimilarityMeasure.ADAMIC_ADAR:
        for d in degs.tolist():
            if d > 1:
                total += 1.0 / math.log(d)
        return total
    for d in degs.tolist():
        if d > 0:
            total += 1.0 / d
    return total


@dataclass
class ClusterResult:
    kept_edges: np.ndarray
    cluster_count: int
    singleton_count: int


def jarvis_patrick_cluster(graph: CsrGraph, provider: IntersectionProvider,
                           tau: float, threads: int = 1) -> ClusterResult:
    """Keep edges whose score strictly exceeds tau; count components.

    Scores, the keep test and the connected components of the kept-edge
    graph (union-find) all run on the device (pg_jp_components); only the
    kept edge list comes back to the host.
    """
    import torch
    graph = as_csr_graph(graph)
    us, vs = graph.device().upper_edges()
    scores = provider._pairs_device(us, vs).to(torch.float64)
    keep = torch.empty(max(1, us.numel()), dtype=torch.uint8, device="cuda")
    out = torch.empty(3, dtype=torch.int64, device="cuda")
    N.call("pg_jp_components", N.ptr(us), N.ptr(vs), N.ptr(scores), us.numel(),
           float(tau), graph.n, N.ptr(keep), N.ptr(out), N.stream_handle())
    kept_n, clusters, touched = (int(x) for x in out.cpu().tolist())
    if kept_n:
        mask = keep[:us.numel()].bool()
        kept = torch.stack([us[mask], vs[mask]], dim=1).cpu().numpy().astype(np.int64)
    else:
        kept = np.empty((0, 2), np.int64)
    return ClusterResult(kept, clusters, graph.n - touched)


@dataclass
class JaccardCount:
    kept_hat: int          # edges with J-hat = m/k >= tau  (est_jaccard_minhash)
    kept_similarity: int   # edges with vertex_similarity(JACCARD) >= tau
    match_hist: np.ndarray  # int64[k+1] edges per positional-match count
    min_matches: int


def jaccard_min_matches(k: int, tau: float) -> int:
    """Smallest m with float32(m)/float32(k) >= float32(tau) (fp32 J-hat)."""
    kf, tf = np.float32(k), np.float32(tau)
    for m in range(k + 1):
        if np.float32(m) / kf >= tf:
            return m
    return k + 1


def jaccard_counts(graph: CsrGraph, sketched: SketchedGraph, tau: float,
                   rank: int = 0, world: int = 1):
    """Device int64 [kept_hat, kept_similarity, match_hist(k+1)] of this
    rank's share of the edge slots."""
    import torch
    from .providers import MinHashProvider
    from .sharding import edge_range
    graph, sketched = as_csr_graph(graph), as_sketched_graph(sketched)
    if sketched.kind is not SketchKind.KHASH:
        raise ValueError("Jaccard clustering needs k-Hash sketches")
    k = sketched.capacity
    d = sketched.device_tensors()
    dev = graph.device()
    us, vs, slots, padded = MinHashProvider(sketched)._tc_layout(dev)
    b, e = edge_range(slots, rank, world, align=32 if padded else 1)
    out = torch.empty(k + 3, dtype=torch.int64, device="cuda")
    N.call("pg_jaccard_count_khash", N.ptr(d["entries"]), k, N.ptr(dev.degrees),
           N.ptr(us), N.ptr(vs), b, e, int(padded), jaccard_min_matches(k, tau),
           float(tau), N.ptr(out), N.stream_handle())
    return out


def jaccard_cluster_count(graph: CsrGraph, sketched: SketchedGraph,
                          tau: float = 0.1) -> JaccardCount:
    """Config 4: per-edge k-Hash Jaccard, kept if >= tau, surviving count."""
    c = jaccard_counts(graph, sketched, tau).cpu().numpy()
    return JaccardCount(int(c[0]), int(c[1]), c[2:].copy(),
                        jaccard_min_matches(sketched.capacity, tau))


# ---------------------------------------------------------------------------
# link prediction (reference mining.py:248-331)


@dataclass
class LinkPredSplit:
    """A disjoint split E = E_sparse + E_removed for prediction testing."""

    sparse_graph: CsrGraph
    edges_sparse: np.ndarray
    edges_removed: np.ndarray
    fraction: float
    seed: int


def make_link_prediction_split(graph: CsrGraph, fraction: float,
                               seed: int) -> LinkPredSplit:
    """Remove round(fraction * m) random edges as the prediction targets.

    The edge sample is the reference's own numpy draw (default_rng(seed)
    .choice without replacement, :262-268) so splits are identical; the
    sparse graph is rebuilt on the device (CsrGraph.from_edges).
    """
    if not 0 <= fraction <= 1:
        raise ValueError("fraction must be in [0, 1]")
    edges = graph.edges()
    rng = np.random.default_rng(seed)
    r = int(round(fraction * len(edges)))
    removed_idx = np.sort(rng.choice(len(edges), size=r, replace=False))
    mask = np.zeros(len(edges), dtype=bool)
    mask[removed_idx] = True
    removed = edges[mask]
    sparse = edges[~mask]
    sparse_graph = CsrGraph.from_edges(sparse, n=graph.n)
    return LinkPredSplit(sparse_graph, sparse, removed, fraction, seed)


def _two_hop_keys(graph: CsrGraph):
    """Device uint64 keys u*n+v (ascending) of the non-adjacent 2-hop pairs."""
    import ctypes
    import torch
    dev = graph.device()
    total = ctypes.c_int64()
    N.call("pg_two_hop_candidates", N.ptr(dev.offsets), N.ptr(dev.adj), graph.n, None, 0,
           ctypes.byref(total), N.stream_handle())
    keys = torch.empty(max(1, total.value), dtype=torch.int64, device="cuda")
    got = ctypes.c_int64()
    N.call("pg_two_hop_candidates", N.ptr(dev.offsets), N.ptr(dev.adj), graph.n,
           N.ptr(keys), keys.numel(), ctypes.byref(got), N.stream_handle())
    return keys[:got.value]


def _two_hop_candidates(graph: CsrGraph) -> np.ndarray:
    """Non-adjacent vertex pairs with at least one common neighbor, (u, v)
    ascending (reference :275-296), computed on the device."""
    if graph.n == 0:
        return np.empty((0, 2), dtype=np.int64)
    k = _two_hop_keys(graph).cpu().numpy()
    return np.stack([k // graph.n, k % graph.n], axis=1).astype(np.int64) if len(k) \
        else np.empty((0, 2), dtype=np.int64)


_MEASURE_CODE = {SimilarityMeasure.JACCARD: 0, SimilarityMeasure.OVERLAP: 1,
                 SimilarityMeasure.COMMON_NEIGHBORS: 2, SimilarityMeasure.TOTAL_NEIGHBORS: 3,
                 SimilarityMeasure.ADAMIC_ADAR: 4, SimilarityMeasure.RESOURCE_ALLOCATION: 5}


def _member_terms(graph: CsrGraph, measure: SimilarityMeasure) -> np.ndarray:
    """term[d] of a degree-d common member, with the reference's expression
    (math.log / float division on the host, so device sums match)."""
    dmax = int(graph.degrees().max()) if graph.n else 0
    t = np.zeros(dmax + 1, dtype=np.float64)
    for d in range(1, dmax + 1):
        if measure is SimilarityMeasure.ADAMIC_ADAR:
            t[d] = 1.0 / math.log(d) if d > 1 else 0.0
        else:
            t[d] = 1.0 / d
    return t


def similarity_scores(graph: CsrGraph, keys, measure, provider: IntersectionProvider):
    """vertex_similarity for a device batch of candidate keys u*n+v."""
    import torch
    from .providers import MinHashProvider
    measure = SimilarityMeasure(measure)
    dev = graph.device()
    count = keys.numel()
    scores = torch.empty(max(1, count), dtype=torch.float64, device="cuda")
    code = _MEASURE_CODE[measure]
    if measure in _COUNTING:
        us = (keys // graph.n).to(torch.int32)
        vs = (keys % graph.n).to(torch.int32)
        est = provider._pairs_device(us, vs).to(torch.float64).contiguous()
        N.call("pg_similarity_scores", code, N.ptr(keys), count, graph.n, N.ptr(dev.offsets),
               N.ptr(est), 0, None, 0, None, None, N.ptr(scores), N.stream_handle())
        return scores[:count]
    term = torch.from_numpy(_member_terms(graph, measure)).cuda()
    if isinstance(provider, ExactProvider):
        src, rows, k, lengths = 0, dev.adj, 0, None
    elif isinstance(provider, MinHashProvider):
        d = provider.sketched.device_tensors()
        rows, k = d["entries"], provider.sketched.capacity
        src, lengths = (1, d["lengths"]) if provider.onehash else (2, None)
    else:
        raise UnsupportedCombinationError(
            f"{provider.kind.value} cannot enumerate intersection members")
    N.call("pg_similarity_scores", code, N.ptr(keys), count, graph.n, N.ptr(dev.offsets),
           None, src, N.ptr(rows), k, N.ptr(lengths) if lengths is not None else None,
           N.ptr(term), N.ptr(scores), N.stream_handle())
    return scores[:count]


def link_prediction_eval(graph: CsrGraph, split: LinkPredSplit,
                         measure, provider: IntersectionProvider,
                         top_count: int) -> int:
    """How many of the top-scored candidate pairs are removed edges.

    Candidates are the 2-hop pairs of the sparse graph; scores come from
    vertex_similarity on the sparse graph; ties rank lexicographically by
    (u, v); ``top_count`` is capped at the candidate count.  The bound
    ``provider`` must be built over ``split.sparse_graph``.  Candidates,
    scores, ranking and the hit count all run on the device.
    """
    import torch
    if len(split.edges_sparse) + len(split.edges_removed) != graph.m:
        raise ValueError("split does not cover the graph's edge set")
    measure = SimilarityMeasure(measure)
    if top_count <= 0:
        return 0
    sparse = split.sparse_graph
    if sparse.n == 0:
        return 0
    keys = _two_hop_keys(sparse)
    if keys.numel() == 0:
        return 0
    scores = similarity_scores(sparse, keys, measure, provider)
    rem = np.asarray(split.edges_removed, dtype=np.int64).reshape(-1, 2)
    removed = np.sort(rem[:, 0] * sparse.n + rem[:, 1])
    removed_d = torch.from_numpy(removed).cuda() if len(removed) else \
        torch.empty(1, dtype=torch.int64, device="cuda")
    hits = torch.empty(1, dtype=torch.int64, device="cuda")
    N.call("pg_rank_top_hits", N.ptr(keys), N.ptr(scores), keys.numel(), int(top_count),
           N.ptr(removed_d), len(removed), N.ptr(hits), N.stream_handle())
    return int(hits.item())


# ---------------------------------------------------------------------------
# sampling baselines for TC (reference mining.py:334-367)


def doulion_tc(graph: CsrGraph, keep_prob: float, seed: int,
               threads: int = 1) -> float:
    """Keep each edge with probability p, count exactly, rescale by p^-3.

    The edge sample is the reference's own draw (default_rng(seed).random
    over graph.edges()); the subgraph, its degree ordering and the exact
    count run on the device.
    """
    if not 0 < keep_prob <= 1:
        raise ValueError("keep probability must be in (0, 1]")
    edges = graph.edges()
    rng = np.random.default_rng(seed)
    kept = edges[rng.random(len(edges)) < keep_prob] if keep_prob < 1 else edges
    sub = CsrGraph.from_edges(kept, n=graph.n)
    view = degree_order(sub)
    exact = ExactProvider.for_view(view)
    return triangle_count(view, exact, threads) / keep_prob ** 3


def reduced_execution_tc(view: DirectedView, fraction: float, seed: int,
                         threads: int = 1) -> float:
    """Node-iterator outer loop over a random vertex subset (the reference's
    default_rng(seed).choice draw), rescaled by 1/fraction; the sampled
    vertices' directed edges are selected and counted exactly on the device."""
    import torch
    if not 0 < fraction <= 1:
        raise ValueError("fraction must be in (0, 1]")
    rng = np.random.default_rng(seed)
    count = max(1, int(round(fraction * view.n)))
    sample = np.sort(rng.choice(view.n, size=count, replace=False))
    dev = view.device()
    if dev.nnz == 0:
        return 0.0
    picked = torch.zeros(view.n, dtype=torch.bool, device="cuda")
    picked[torch.from_numpy(sample).cuda()] = True
    src = dev.row_sources()
    sel = picked[src.long()]
    exact = ExactProvider.for_view(view)
    total = exact._pairs_device(src[sel].contiguous(), dev.adj[sel].contiguous())
    return float(int(total.sum().item()) if total.numel() else 0) / fraction
