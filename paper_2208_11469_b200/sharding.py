"""Edge-range sharding across the GPUs of one node.

Every rank holds the full sketch matrix (replicated: 4 GiB at config 5 is
small next to 180 GB of HBM) and processes one contiguous range of the
upper-triangular edge list.  The per-edge statistics of the fused kernels
are exact integers (popcount histograms, per-match-count sums), so one
``all_reduce(SUM)`` of that small vector over NCCL yields exactly the
single-GPU result for any world size; KMV is the only fp64 partial.

The host logic (ranges, reduction, combination) is independent of the
device and is exercised with the gloo backend on CPU in tests.
"""

from __future__ import annotations

import numpy as np

__all__ = ["edge_range", "weighted_edge_range", "allreduce_counts",
           "tc_estimate_sharded", "four_clique_count_sharded"]


def edge_range(m: int, rank: int, world: int, align: int = 1) -> tuple[int, int]:
    """Contiguous, balanced [begin, end) share of m edge slots for ``rank``;
    interior boundaries are multiples of ``align`` (padded layouts)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if align > 1:
        units = (m + align - 1) // align
        b, e = edge_range(units, rank, world)
        return min(b * align, m), min(e * align, m)
    base, extra = divmod(m, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def weighted_edge_range(weights_prefix: np.ndarray, rank: int,
                        world: int) -> tuple[int, int]:
    """Split by equal shares of a work prefix sum (4-clique: d+u + d+v)."""
    total = int(weights_prefix[-1]) if len(weights_prefix) else 0
    lo = np.searchsorted(weights_prefix, total * rank / world, side="left")
    hi = np.searchsorted(weights_prefix, total * (rank + 1) / world, side="left")
    if rank == world - 1:
        hi = len(weights_prefix)
    return int(lo), int(hi)


def allreduce_counts(counts, group=None):
    """SUM-allreduce of a partial-count tensor (NCCL on GPU, gloo on CPU)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def tc_estimate_sharded(graph, sketched=None, kind="bf_and", group=None):
    """tc_estimate over this rank's edge range + one allreduce."""
    import torch.distributed as dist
    from .mining import _tc_provider, tc_combine, tc_counts
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    provider = _tc_provider(graph, sketched, kind)
    counts = allreduce_counts(tc_counts(provider, graph.device(), rank, world), group)
    return tc_combine(provider, counts.cpu().numpy()) / 3.0


def four_clique_count_sharded(view, provider, group=None):
    import torch.distributed as dist
    from .mining import four_clique_combine, four_clique_counts
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    outdeg = view.out_degrees()
    src = np.repeat(np.arange(view.n, dtype=np.int64), outdeg)
    work = np.cumsum(outdeg[src] + outdeg[view.adjacency])
    b, e = weighted_edge_range(work, rank, world)
    counts = allreduce_counts(four_clique_counts(view, provider, b, e), group)
    return four_clique_combine(provider, counts.cpu().numpy())
