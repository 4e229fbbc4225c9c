"""Estimator kinds, the Swamidass table and the per-pair scalar estimators.

Restates reference ``estimators.py``: ``EstimatorKind`` (:54-62),
``swamidass_value`` (:65-70), ``est_single_*`` (:73-86) and the pairwise
estimators (:95-200).  The pairwise functions take host sketch records like
the reference, but their integer core (popcount of AND/OR, positional or set
matches, KMV union statistics) is computed by the device kernels through a
two-row batch; only the O(1) closed-form tail runs on the host.

``swamidass_table(B, b)`` evaluates ``swamidass_value`` for every possible
popcount 0..B with numpy's ``log1p`` -- the same expression the reference
evaluates per edge -- so a per-edge table lookup on the device is
bit-identical to the reference's per-edge value.
"""

from __future__ import annotations

import enum
import threading
from functools import lru_cache

import numpy as np

from .sketches import BloomSketch, KHashSketch, KmvSketch, OneHashSketch

__all__ = ["EstimatorKind", "swamidass_value", "swamidass_table",
           "est_single_swamidass", "est_single_delta_class",
           "est_intersection_bf_and", "est_intersection_bf_limit",
           "est_intersection_bf_or", "est_jaccard_minhash",
           "est_intersection_minhash", "est_intersection_kmv"]


class EstimatorKind(str, enum.Enum):
    EXACT_MERGE = "exact_merge"
    EXACT_GALLOP = "exact_gallop"
    BF_AND = "bf_and"
    BF_L = "bf_l"
    BF_OR = "bf_or"
    KHASH = "khash"
    ONEHASH = "onehash"
    KMV = "kmv"


def swamidass_value(bit_length, hash_count, ones):
    """-(B/b) * log1p(-(ones - [ones == B]) / B); array friendly."""
    o = np.asarray(ones, dtype=np.float64)
    o_adj = o - (o == bit_length)
    val = -(bit_length / hash_count) * np.log1p(-o_adj / bit_length)
    return val if val.ndim else float(val)


@lru_cache(maxsize=64)
def _table(bits: int, b: int) -> np.ndarray:
    t = swamidass_value(bits, b, np.arange(bits + 1, dtype=np.float64))
    t = np.ascontiguousarray(t, dtype=np.float64)
    t.setflags(write=False)
    return t


def swamidass_table(bits: int, b: int) -> np.ndarray:
    """float64[bits+1]: the estimate of every possible popcount."""
    return _table(int(bits), int(b))


def est_single_swamidass(sketch: BloomSketch) -> float:
    return swamidass_value(sketch.bit_length, sketch.hash_count, sketch.ones)


def est_single_delta_class(ones: int, delta: float) -> float:
    if delta < 0:
        raise ValueError("delta must be >= 0")
    return float(delta * ones)


# ---------------------------------------------------------------------------
# two-row device batches


_STAGE = threading.local()


class _Pinned:
    """Per-thread pinned (device-mapped) staging for the two-row scalar
    estimators: the rows, the edge (0, 1), the sizes and the outputs sit in
    one host buffer the kernel reads and writes directly -- one launch and
    one stream synchronisation per call, no device allocations or copies."""

    def __init__(self, rows: np.ndarray, n_out: int):
        import torch
        rows = np.ascontiguousarray(rows)
        need = rows.nbytes + 16 + 8 + 8 * n_out + 64
        buf = getattr(_STAGE, "buf", None)
        if buf is None or buf.numel() < need:
            buf = _STAGE.buf = torch.empty(max(need, 1 << 16), dtype=torch.uint8, pin_memory=True)
        self.base = buf.data_ptr()
        host = buf.numpy()
        host[:rows.nbytes] = rows.view(np.uint8).reshape(-1)
        self.rows = self.base
        o = (rows.nbytes + 15) & ~15
        ids = host[o:o + 8].view(np.int32)
        ids[0], ids[1] = 0, 1
        self.us, self.vs = self.base + o, self.base + o + 4
        self.sizes_host = host[o + 8:o + 16].view(np.int32)
        self.sizes = self.base + o + 8
        self.out_host = host[o + 16:o + 16 + 8 * n_out].view(np.int64)
        self.outs = [self.base + o + 16 + 8 * i for i in range(n_out)]
        self.out_host[:] = 0

    def sync(self):
        import torch
        torch.cuda.current_stream().synchronize()


def _bloom_count(sx: BloomSketch, sy: BloomSketch, use_or: bool) -> int:
    from . import _native as N
    if (sx.bit_length != sy.bit_length or sx.hash_count != sy.hash_count
            or sx.seed != sy.seed):
        raise ValueError("Bloom sketches have mismatched parameters")
    rows = np.stack([np.asarray(sx.words, dtype=np.uint64),
                     np.asarray(sy.words, dtype=np.uint64)])
    st = _Pinned(rows, 1)
    op = N.PG_BF_OR if use_or else N.PG_BF_AND
    N.call("pg_pairs_bloom", st.rows, sx.bit_length, sx.hash_count, op, None,
           None, st.us, st.vs, 1, st.outs[0], None, N.stream_handle())
    st.sync()
    return int(st.out_host[0:1].view(np.int32)[0])


def est_intersection_bf_and(sx: BloomSketch, sy: BloomSketch) -> float:
    return swamidass_value(sx.bit_length, sx.hash_count, _bloom_count(sx, sy, False))


def est_intersection_bf_limit(sx: BloomSketch, sy: BloomSketch) -> float:
    return _bloom_count(sx, sy, False) / sx.hash_count


def est_intersection_bf_or(sx: BloomSketch, sy: BloomSketch, size_x: int,
                           size_y: int, clamp: bool = True) -> float:
    ones = _bloom_count(sx, sy, True)
    raw = size_x + size_y - swamidass_value(sx.bit_length, sx.hash_count, ones)
    return max(0.0, raw) if clamp else raw


def _padded_ids(entries: np.ndarray, k: int) -> np.ndarray:
    row = np.full(k, -1, dtype=np.int32)
    e = np.asarray(entries, dtype=np.int64)
    row[:len(e)] = e
    return row


def _minhash_matches(mx, my, onehash: bool) -> int:
    import torch
    from . import _native as N
    k = mx.capacity
    rows = np.stack([_padded_ids(mx.entries, k), _padded_ids(my.entries, k)])
    st = _Pinned(rows, 1)
    st.sizes_host[0], st.sizes_host[1] = len(mx.entries), len(my.entries)
    N.call("pg_pairs_minhash", st.rows, k, int(onehash), st.sizes, st.us, st.vs, 1,
           st.outs[0], None, N.stream_handle())
    st.sync()
    return int(st.out_host[0:1].view(np.int32)[0])


def est_jaccard_minhash(mx, my) -> float:
    if isinstance(mx, KHashSketch) and isinstance(my, KHashSketch):
        if mx.capacity != my.capacity:
            raise ValueError("k-Hash sketches have mismatched k")
        if len(mx.entries) == 0 or len(my.entries) == 0:
            return 0.0
        return _minhash_matches(mx, my, False) / mx.capacity
    if isinstance(mx, OneHashSketch) and isinstance(my, OneHashSketch):
        if mx.capacity != my.capacity:
            raise ValueError("1-Hash sketches have mismatched k")
        lx, ly = len(mx.entries), len(my.entries)
        if lx == 0 and ly == 0:
            return 0.0
        common = _minhash_matches(mx, my, True) if lx and ly else 0
        denom = min(mx.capacity, lx + ly - common)
        return common / denom if denom else 0.0
    raise TypeError("need two k-Hash or two 1-Hash sketches of equal kind")


def est_intersection_minhash(mx, my, size_x: int, size_y: int) -> float:
    if isinstance(mx, OneHashSketch) and isinstance(my, OneHashSketch):
        if mx.capacity != my.capacity:
            raise ValueError("1-Hash sketches have mismatched k")
        if size_x <= mx.capacity and size_y <= my.capacity:
            if len(mx.entries) == 0 or len(my.entries) == 0:
                return 0.0
            return float(_minhash_matches(mx, my, True))
    j = est_jaccard_minhash(mx, my)
    return (j / (1.0 + j)) * (size_x + size_y)


def kmv_union_stats(kx: KmvSketch, ky: KmvSketch):
    """(common, union, k_eff, kth) of two KMV sketches, from the device."""
    import torch
    from . import _native as N
    if kx.capacity != ky.capacity:
        raise ValueError("KMV sketches have mismatched k")
    k = kx.capacity
    rows = np.full((2, k), np.inf, dtype=np.float64)
    rows[0, :len(kx.hashes)] = kx.hashes
    rows[1, :len(ky.hashes)] = ky.hashes
    st = _Pinned(rows, 3)
    st.sizes_host[:] = 0
    N.call("pg_pairs_kmv", st.rows, None, k, st.sizes, st.us, st.vs, 1, st.outs[0],
           st.outs[1], st.outs[2], None, N.stream_handle())
    st.sync()
    return (int(st.out_host[0:1].view(np.int32)[0]), int(st.out_host[1:2].view(np.int32)[0]),
            min(len(kx.hashes), len(ky.hashes)), float(st.out_host[2:3].view(np.float64)[0]))


def est_intersection_kmv(kx: KmvSketch, ky: KmvSketch, size_x: int,
                         size_y: int, clamp: bool = True) -> float:
    common, union, k_eff, kth = kmv_union_stats(kx, ky)
    cap = kx.capacity
    if size_x <= cap and size_y <= cap:
        raw = float(size_x + size_y - union)
    elif k_eff < 2:
        raw = float(common)
    else:
        raw = size_x + size_y - (k_eff - 1) / kth
    if not clamp:
        return raw
    return float(min(max(raw, 0.0), min(size_x, size_y)))
