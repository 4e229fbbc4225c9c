"""Intersection providers: the plugin surface the mining drivers call.

Same names, signatures and errors as reference ``providers.py``
(``IntersectionProvider`` :44-64, ``ExactProvider`` :67-121,
``BloomProvider`` :124-175, ``MinHashProvider`` :178-250, ``KmvProvider``
:253-307, ``make_provider`` :310-338).  Every batch call runs the sm_100a
kernels of the C ABI:

  * ``pair_many(us, vs)`` accepts host numpy arrays (returns numpy, like the
    reference) or int CUDA tensors (returns a float64 CUDA tensor, no host
    round trip);
  * ``_tc_counts(e_begin, e_end)`` is the fused whole-graph pass used by
    ``tc_estimate`` (integer outputs, combined on the host by
    ``_tc_combine``), also per edge shard for the multi-GPU driver.

Providers are read-only after construction; concurrent ``pair_many`` calls
from several threads each allocate their own buffers and enqueue on the
current stream, which is safe.
"""

from __future__ import annotations

import math
import threading

import numpy as np

from . import _native as N
from .estimators import (EstimatorKind, est_intersection_kmv,
                         est_intersection_minhash, swamidass_table,
                         swamidass_value)
from .graphs import CsrGraph, DeviceCsr, DirectedView
from .graphs import as_csr_graph, as_directed_view
from .sketches import (SketchKind, SketchedGraph, as_sketched_graph, build_bloom,
                       build_khash, build_kmv, build_onehash)

__all__ = ["UnsupportedCombinationError", "IntersectionProvider",
           "ExactProvider", "BloomProvider", "MinHashProvider", "KmvProvider",
           "make_provider"]


class UnsupportedCombinationError(ValueError):
    """Asked a provider for something its sketch kind cannot deliver."""


def _as_device_ids(a, n: int | None = None):
    """int32 device vertex IDs.  With n given, indices follow numpy's rules
    as the reference's row gathers do: -n <= i < 0 wraps, anything outside
    [-n, n) raises IndexError -- the kernels never see an out-of-range row."""
    import torch
    if isinstance(a, torch.Tensor):
        t = a.to(device="cuda", dtype=torch.int64).reshape(-1)
        if n is not None and t.numel():
            lo, hi = int(t.min().item()), int(t.max().item())
            if lo < -n or hi >= n:
                bad = hi if hi >= n else lo
                raise IndexError(f"index {bad} is out of bounds for axis 0 with size {n}")
            if lo < 0:
                t = torch.where(t < 0, t + n, t)
        return t.to(torch.int32).contiguous(), True
    arr = np.asarray(a, dtype=np.int64).reshape(-1)
    if n is not None and arr.size:
        lo, hi = int(arr.min()), int(arr.max())
        if lo < -n or hi >= n:
            bad = hi if hi >= n else lo
            raise IndexError(f"index {bad} is out of bounds for axis 0 with size {n}")
        if lo < 0:
            arr = np.where(arr < 0, arr + n, arr)
    return torch.from_numpy(arr.astype(np.int32)).cuda(), False


_SCALAR = threading.local()


def _scalar_staging():
    """Per-thread pinned (device-mapped) buffers for the scalar calls: the
    two IDs go in and the result comes back without device allocations or
    copy launches -- the kernel reads and writes them over the mapped
    pointers, and one stream synchronisation ends the call."""
    st = getattr(_SCALAR, "buf", None)
    if st is None:
        import torch
        ids = torch.empty(2, dtype=torch.int32, pin_memory=True)
        out = torch.empty(2, dtype=torch.int64, pin_memory=True)
        st = _SCALAR.buf = (ids, ids.numpy(), out, out.numpy())
    return st


def _row_index(i, n: int) -> int:
    """numpy's row-index rules, as the reference's row gathers."""
    i = int(i)
    if i < -n or i >= n:
        raise IndexError(f"index {i} is out of bounds for axis 0 with size {n}")
    return i + n if i < 0 else i


class IntersectionProvider:
    kind: EstimatorKind
    is_exact = False

    def pair(self, u: int, v: int) -> float:
        """One edge's estimate: the batch kernel on one slot, with the IDs
        and the result in pinned mapped memory (one launch + one stream
        synchronisation, no allocations)."""
        import torch
        n = self._num_vertices()
        u, v = _row_index(u, n), _row_index(v, n)
        ids_t, ids, out_t, out = _scalar_staging()
        ids[0], ids[1] = u, v
        self._pairs_launch(ids_t.data_ptr(), ids_t.data_ptr() + 4, 1, out_t.data_ptr())
        torch.cuda.current_stream().synchronize()
        if self.is_exact:
            return int(out[0])
        return float(out.view(np.float64)[0])

    def _pairs_launch(self, us_ptr: int, vs_ptr: int, count: int, out_ptr: int) -> None:
        """Enqueue the per-edge kernel over raw pointers (device or mapped)."""
        raise NotImplementedError

    def _num_vertices(self) -> int:
        raise NotImplementedError

    def pair_many(self, us, vs):
        n = self._num_vertices()
        du, on_dev = _as_device_ids(us, n)
        dv, _ = _as_device_ids(vs, n)
        if du.shape != dv.shape:
            raise ValueError("us and vs must have the same length")
        out = self._pairs_device(du, dv)
        return out if on_dev else out.cpu().numpy()

    def _pairs_device(self, us, vs):
        raise NotImplementedError

    def with_set(self, w: int, members) -> float:
        raise NotImplementedError

    def common_members(self, u: int, v: int) -> np.ndarray:
        raise UnsupportedCombinationError(
            f"{self.kind.value} cannot enumerate intersection members")


class ExactProvider(IntersectionProvider):
    """Exact |N(u) & N(v)| from sorted CSR rows, on the device."""

    is_exact = True

    def __init__(self, offsets, adjacency, strategy: str = "merge"):
        if strategy not in ("merge", "gallop", "auto"):
            raise ValueError("strategy must be merge, gallop, or auto")
        self.offsets = np.asarray(offsets, dtype=np.int64)
        self.adjacency = np.asarray(adjacency, dtype=np.int64)
        self.strategy = strategy
        self.sizes = np.diff(self.offsets)
        self.kind = (EstimatorKind.EXACT_GALLOP if strategy == "gallop"
                     else EstimatorKind.EXACT_MERGE)
        self._dev = None

    @classmethod
    def for_graph(cls, graph: CsrGraph, strategy: str = "merge"):
        p = cls(graph.offsets, graph.adjacency, strategy)
        p._dev = graph.device()
        return p

    @classmethod
    def for_view(cls, view: DirectedView, strategy: str = "merge"):
        p = cls(view.offsets, view.adjacency, strategy)
        p._dev = view.device()
        return p

    def device(self) -> DeviceCsr:
        if self._dev is None:
            self._dev = DeviceCsr(self.offsets, self.adjacency)
        return self._dev

    def _num_vertices(self) -> int:
        return len(self.offsets) - 1

    def _pairs_launch(self, us_ptr, vs_ptr, count, out_ptr):
        d = self.device()
        N.call("pg_pairs_exact", N.ptr(d.offsets), N.ptr(d.adj), us_ptr, vs_ptr, count,
               out_ptr, N.stream_handle())

    def _pairs_device(self, us, vs):
        import torch
        out = torch.empty(max(1, us.numel()), dtype=torch.int64, device="cuda")
        self._pairs_launch(N.ptr(us), N.ptr(vs), us.numel(), N.ptr(out))
        return out[:us.numel()]

    def with_set(self, w: int, members) -> int:
        m = np.unique(np.asarray(members, dtype=np.int64))
        return int(np.count_nonzero(np.isin(
            self.adjacency[self.offsets[w]:self.offsets[w + 1]], m,
            assume_unique=True)))

    def common_members(self, u: int, v: int) -> np.ndarray:
        a = self.adjacency[self.offsets[u]:self.offsets[u + 1]]
        b = self.adjacency[self.offsets[v]:self.offsets[v + 1]]
        return np.intersect1d(a, b, assume_unique=True)


class TcLayout:
    """Edge slots of a fused whole-graph pass: (us, vs, slots, padded)
    unpack like a tuple; ``kind`` names the schedule ("id": every edge u < v
    in CSR order; "hub": degree-oriented with hub tags, ``hub_ids``)."""

    __slots__ = ("us", "vs", "slots", "padded", "kind", "hub_ids", "n_hubs", "split", "regroup")

    def __init__(self, us, vs, slots, padded, kind="id", hub_ids=None, n_hubs=0, split=None, regroup=0):
        self.us, self.vs, self.slots, self.padded = us, vs, slots, padded
        self.kind, self.hub_ids, self.n_hubs = kind, hub_ids, n_hubs
        self.regroup = regroup  # degree layout: N+ rows of <= regroup entries grouped by their other endpoint
        self.split = split  # KMV merge layout: slots [0, split) stop after k_eff steps

    def __iter__(self):
        return iter((self.us, self.vs, self.slots, self.padded))

    def __getitem__(self, i):
        return (self.us, self.vs, self.slots, self.padded)[i]


_WITH_SET_CAP = 2048  # members the one-warp with_set kernel holds (pg_scalar.cu)


class _SketchProvider(IntersectionProvider):
    def __init__(self, sketched: SketchedGraph):
        self.sketched = as_sketched_graph(sketched)

    def _with_set_device(self, w, members, code: int, width: int, lut=None):
        """with_set in one launch (pg_with_set): the members go to the
        device sorted, repeats kept, through a pinned mapped buffer.
        None when the set or the sketch exceeds the one-warp kernel (the
        caller then builds the member sketch with the batch builders)."""
        import torch
        sg = self.sketched
        raw = np.sort(np.asarray(members, dtype=np.int64).reshape(-1))
        w = _row_index(w, sg.n)
        if len(raw) and (raw[0] < 0 or raw[-1] >= 2 ** 31):
            raise ValueError("set members must be int32 vertex IDs")
        if len(raw) > _WITH_SET_CAP:
            return None
        st = getattr(_SCALAR, "set", None)
        if st is None:
            mt = torch.empty(_WITH_SET_CAP, dtype=torch.int32, pin_memory=True)
            ot = torch.empty(1, dtype=torch.float64, pin_memory=True)
            st = _SCALAR.set = (mt, mt.numpy(), ot, ot.numpy())
        mt, mv, ot, ov = st
        mv[:len(raw)] = raw
        d = self._dev()
        rows = d.get("rows") if "rows" in d else d.get("values", d.get("entries"))
        lengths = d.get("lengths")
        rc = N.lib().pg_with_set(code, N.ptr(rows), N.ptr(lengths) if lengths is not None else None,
                                 N.ptr(d["sizes"]), width, sg.hash_count, N.ptr(d["seeds"]),
                                 N.ptr(lut) if lut is not None else None, w, mt.data_ptr(),
                                 len(raw), ot.data_ptr(), N.stream_handle())
        if rc == N.PG_ERR_UNSUPPORTED:
            return None
        N.check(rc, "pg_with_set")
        torch.cuda.current_stream().synchronize()
        return float(ov[0])

    @property
    def sizes(self) -> np.ndarray:
        return self.sketched.sizes

    def tc_pad(self) -> int:
        """Lane-group size of the fused kernel = pad of its edge-slot layout."""
        return 1

    def _tc_layout(self, dev):
        """(us, vs, slots, padded) edge-slot arrays the fused kernel consumes."""
        pad = self.tc_pad()
        if pad > 1:
            us, vs, slots = dev.upper_edges_padded(pad)
            return TcLayout(us, vs, slots, True)
        us, vs = dev.upper_edges()
        return TcLayout(us, vs, us.numel(), False)

    def _tc_counts_layout(self, lay, e_begin: int, e_end: int):
        """The fused pass over slots [e_begin, e_end) of a _tc_layout."""
        return self._tc_counts(lay.us, lay.vs, e_begin, e_end, lay.padded)

    def _tc_counts_shard(self, lay, rank: int, world: int):
        """This rank's share of a _tc_layout: a contiguous, balanced slot
        range (sharding.edge_range; padded layouts split on 32-slot units)."""
        from .sharding import edge_range
        b, e = edge_range(lay.slots, rank, world, align=32 if lay.padded else 1)
        return self._tc_counts_layout(lay, b, e)

    @staticmethod
    def _tc_layout_name(lay) -> str:
        if lay.kind == "hub":
            return (f"degree-oriented group-u slots (pad 8), {lay.n_hubs} hub rows staged "
                    "in shared memory per CTA")
        if lay.kind == "degree":
            name = ("degree-oriented row-padded slots (u = lower (degree, ID) rank, N+ lists "
                    "of degree_order), one u per slot group")
            if lay.regroup > 0:
                name += (f"; last slot groups of <= {lay.regroup} entries regrouped by their "
                         "higher-rank endpoint (fewer pad slots)")
            return name
        if lay.kind.endswith("+onehash-rank"):
            return ("row-padded slots grouped by the table endpoint ("
                    + ("higher (degree, ID) rank" if lay.kind.startswith("degree") else "lower ID")
                    + "), each row sorted by its probe count")
        if lay.kind.endswith("+kmv-merge"):
            return ("every edge once, " + ("lower -> higher (degree, ID) rank" if lay.kind.startswith("degree")
                                          else "u < v") + ", partitioned [k_eff-step merges | full merges]")
        return {0: "upper edges u < v (CSR order)", 1: "row-padded upper edges",
                2: "row-padded upper edges, one u per slot group"}[int(lay.padded)]

    def _dev(self) -> dict:
        return self.sketched.device_tensors()

    def _num_vertices(self) -> int:
        return self.sketched.n


_LUTS = {}


def _device_lut(bits: int, b: int):
    """The Swamidass table on the current device, uploaded once per (B, b):
    a per-provider pageable upload would stall the host before every pass."""
    import torch
    key = (bits, b, torch.cuda.current_device())
    if key not in _LUTS:
        _LUTS[key] = torch.from_numpy(swamidass_table(bits, b).copy()).cuda()
    return _LUTS[key]


class BloomProvider(_SketchProvider):
    """Bloom estimates; ``kind`` picks the AND, limit or OR form."""

    def __init__(self, sketched: SketchedGraph, kind: EstimatorKind):
        sketched = as_sketched_graph(sketched)
        if sketched.kind is not SketchKind.BLOOM:
            raise ValueError("BloomProvider needs Bloom sketches")
        kind = EstimatorKind(getattr(kind, "value", kind))
        if kind not in (EstimatorKind.BF_AND, EstimatorKind.BF_L,
                        EstimatorKind.BF_OR):
            raise ValueError(f"{kind} is not a Bloom estimator")
        super().__init__(sketched)
        self.kind = kind
        self._lut = None

    @property
    def op(self) -> int:
        return {EstimatorKind.BF_AND: N.PG_BF_AND, EstimatorKind.BF_L: N.PG_BF_L,
                EstimatorKind.BF_OR: N.PG_BF_OR}[self.kind]

    def lut_device(self):
        if self._lut is None:
            self._lut = _device_lut(self.sketched.bit_length, self.sketched.hash_count)
        return self._lut

    def _pairs_launch(self, us_ptr, vs_ptr, count, out_ptr):
        d, sg = self._dev(), self.sketched
        N.call("pg_pairs_bloom", N.ptr(d["rows"]), sg.bit_length, sg.hash_count, self.op,
               N.ptr(d["sizes"]), N.ptr(self.lut_device()), us_ptr, vs_ptr, count, None,
               out_ptr, N.stream_handle())

    def _pairs_device(self, us, vs):
        import torch
        out = torch.empty(max(1, us.numel()), dtype=torch.float64, device="cuda")
        self._pairs_launch(N.ptr(us), N.ptr(vs), us.numel(), N.ptr(out))
        return out[:us.numel()]

    def pair_counts(self, us, vs):
        """Per-edge popcounts of AND (OR for BF_OR) -- the integer core."""
        import torch
        du, on_dev = _as_device_ids(us, self.sketched.n)
        dv, _ = _as_device_ids(vs, self.sketched.n)
        d, sg = self._dev(), self.sketched
        out = torch.empty(max(1, du.numel()), dtype=torch.int32, device="cuda")
        N.call("pg_pairs_bloom", N.ptr(d["rows"]), sg.bit_length,
               sg.hash_count, self.op, None, None, N.ptr(du), N.ptr(dv),
               du.numel(), N.ptr(out), None, N.stream_handle())
        out = out[:du.numel()]
        return out if on_dev else out.cpu().numpy().astype(np.int64)

    def tc_pad(self) -> int:
        return N.group_pad(self.sketched.bit_length // 8)

    DEGREE_ORIENT_MIN_BYTES = 512 << 20

    def hub_capacity(self) -> int:
        """Hub rows the degree-oriented engine stages per CTA (0: none for
        this row width, or disabled with PG_TC_HUB=0)."""
        import ctypes
        import os
        if os.environ.get("PG_TC_HUB", "0") == "0":
            return 0
        cap = ctypes.c_int32()
        N.call("pg_tc_bloom_hub_capacity", self.sketched.bit_length, ctypes.byref(cap))
        env = os.environ.get("PG_TC_HUBS")
        return min(cap.value, int(env)) if env else cap.value

    def _tc_layout(self, dev):
        """Bloom TC edge schedule.  Row widths with a lane-group engine take
        the row-padded layout with one u per slot group (padded mode 2 of
        pg_tc_bloom), every edge oriented from its lower- to its higher-
        (degree, ID)-rank endpoint (the N+ lists of degree_order): the u row
        held in registers across its run is the low-degree side, and the
        streamed v rows are the hub side, which stays resident in L1/L2
        (PG_TC_ORIENT=id: u < v by ID instead).  PG_TC_HUB=1 selects the
        shared-memory hub engine (pg_tc_bloom_hub, 2048-bit rows).  Every
        per-edge popcount is symmetric in (u, v), so any schedule yields the
        same histogram."""
        import os
        cap = self.hub_capacity()
        if cap > 0 and dev.n > 0:
            n_hubs = min(cap, dev.n)
            ug, vs, slots, hub_ids = dev.hub_slots(8, n_hubs)
            return TcLayout(ug, vs, slots, 2, "hub", hub_ids, n_hubs)
        pad = self.tc_pad()
        if pad > 1:
            # measured (scripts/probe_tc.py): degree orientation wins where
            # the matrix streams from HBM (c5 4 GiB: 5.48 -> 4.70 ms) and
            # loses where it is L2-resident (c2 128 MiB: 0.196 -> 0.21 ms)
            sg = self.sketched
            big = sg.n * sg.bit_length // 8 > self.DEGREE_ORIENT_MIN_BYTES
            orient = os.environ.get("PG_TC_ORIENT", "degree" if big else "id")
            if orient == "degree" and dev.n > 0:
                # a row's last slot group of at most `thr` entries is regrouped
                # by the other endpoint (DeviceCsr.hybrid_slots): 19 % -> 7 % pad
                # slots at R-MAT; c5 4.43 -> 4.11 ms (thr 4; 2: 4.16, 3: 4.12, 5: 4.12)
                thr = int(os.environ.get("PG_TC_HYBRID", "4"))
                if thr > 0 and dev.nnz > 0:
                    ug, vs, slots = dev.hybrid_slots(pad, thr)
                    return TcLayout(ug, vs, slots, 2, "degree", regroup=thr)
                ug, vs, slots, _ = dev.hub_slots(pad, 0)
                return TcLayout(ug, vs, slots, 2, "degree")
            thr = int(os.environ.get("PG_TC_HYBRID_ID", "0"))
            if thr > 0 and dev.nnz > 0:
                ug, vs, slots = dev.hybrid_slots(pad, thr, "id")
                return TcLayout(ug, vs, slots, 2, regroup=thr)
            ug, vs, slots = dev.upper_edges_group_u(pad)
            return TcLayout(ug, vs, slots, 2)
        return super()._tc_layout(dev)

    def _tc_counts_layout(self, lay, e_begin: int, e_end: int):
        if lay.kind != "hub":
            return super()._tc_counts_layout(lay, e_begin, e_end)
        import torch
        d, sg = self._dev(), self.sketched
        out = torch.empty(sg.bit_length + 2, dtype=torch.int64, device="cuda")
        N.call("pg_tc_bloom_hub", N.ptr(d["rows"]), sg.bit_length, self.op,
               N.ptr(d["sizes"]), N.ptr(self.lut_device()), N.ptr(lay.us), N.ptr(lay.vs),
               e_begin, e_end, N.ptr(lay.hub_ids), lay.n_hubs, N.ptr(out),
               N.ptr(out) + 8 * (sg.bit_length + 1), N.stream_handle())
        return out

    def _tc_counts(self, us, vs, e_begin: int, e_end: int, padded: bool = False):
        import torch
        d, sg = self._dev(), self.sketched
        # [hist(B+1) | sum_pos]: one buffer, one memset, no concatenation
        out = torch.empty(sg.bit_length + 2, dtype=torch.int64, device="cuda")
        N.call("pg_tc_bloom", N.ptr(d["rows"]), sg.bit_length, self.op,
               N.ptr(d["sizes"]), N.ptr(self.lut_device()), N.ptr(us), N.ptr(vs),
               e_begin, e_end, int(padded), N.ptr(out), N.ptr(out) + 8 * (sg.bit_length + 1),
               N.stream_handle())
        return out

    def _tc_combine(self, counts: np.ndarray) -> float:
        """Sum of per-edge estimates from the exact integer outputs."""
        sg = self.sketched
        hist, spos = counts[:-1], int(counts[-1])
        if self.kind is EstimatorKind.BF_L:
            return float(int(np.dot(hist, np.arange(len(hist), dtype=np.int64)))
                         / sg.hash_count)
        lut = swamidass_table(sg.bit_length, sg.hash_count)
        nz = np.nonzero(hist)[0]
        # float(hist[o]) * lut[o] per bin (vectorised), exactly-rounded sum
        weighted = math.fsum((hist[nz].astype(np.float64) * lut[nz]).tolist())
        if self.kind is EstimatorKind.BF_AND:
            return weighted
        return float(spos) - weighted

    def with_set(self, w: int, members) -> float:
        sg = self.sketched
        got = self._with_set_device(w, members, self.op, sg.bit_length,
                                    None if self.kind is EstimatorKind.BF_L else self.lut_device())
        if got is not None:
            return got
        members = np.asarray(members, dtype=np.int64)
        mem = build_bloom(members, sg.plan, sg.family)
        from .estimators import _bloom_count
        from .sketches import BloomSketch
        row = sg.sketch(w)
        ones = _bloom_count(row, BloomSketch(mem.words, sg.bit_length,
                                             sg.hash_count, mem.ones, sg.seed),
                            self.kind is EstimatorKind.BF_OR)
        if self.kind is EstimatorKind.BF_OR:
            raw = (int(self.sizes[w]) + len(members)
                   - swamidass_value(sg.bit_length, sg.hash_count, ones))
            return max(0.0, float(raw))
        if self.kind is EstimatorKind.BF_L:
            return ones / sg.hash_count
        return float(swamidass_value(sg.bit_length, sg.hash_count, ones))


class MinHashProvider(_SketchProvider):
    """k-Hash or 1-Hash estimates from entry matrices."""

    def __init__(self, sketched: SketchedGraph):
        sketched = as_sketched_graph(sketched)
        if sketched.kind is SketchKind.KHASH:
            self.kind = EstimatorKind.KHASH
        elif sketched.kind is SketchKind.ONEHASH:
            self.kind = EstimatorKind.ONEHASH
        else:
            raise ValueError("MinHashProvider needs MinHash sketches")
        super().__init__(sketched)

    @property
    def onehash(self) -> bool:
        return self.kind is EstimatorKind.ONEHASH

    def tc_pad(self) -> int:
        k = self.sketched.capacity
        if self.onehash:  # per-warp-table engine: one u per warp iteration
            return N.onehash_block_pad(k)
        return N.group_pad(4 * k)

    def _tc_layout(self, dev):
        """k-Hash rows of 64/128/256 bytes take the degree-oriented group-u
        layout (as BloomProvider._tc_layout) when the entry matrix streams
        from HBM: the register-held u row is then the low-degree endpoint
        and the streamed v rows the hub side, which stays in L2 (with u < v
        by ID, the Chung-Lu hubs at low IDs are the u side and every edge
        misses on its v row).  Positional matches and s_u + s_v are
        symmetric, so the statistics are the same integers.  1-Hash keeps
        its per-warp-table layout; PG_TC_ORIENT=id restores u < v."""
        import os
        sg = self.sketched
        pad = self.tc_pad()
        if self.onehash and pad > 1 and dev.n > 0 and dev.nnz > 0:
            lay = self._onehash_rank_layout(dev, pad)
            if lay is not None:
                return lay
        if (not self.onehash and pad > 1 and sg.capacity in (16, 32, 64) and dev.n > 0
                and sg.n * sg.capacity * 4 > BloomProvider.DEGREE_ORIENT_MIN_BYTES
                and os.environ.get("PG_TC_ORIENT", "degree") == "degree"):
            # as BloomProvider: nearly empty last slot groups regrouped by the
            # other endpoint (c4: 2.749 -> 2.712 ms at 2; 1: 2.726)
            thr = int(os.environ.get("PG_TC_HYBRID_KHASH", "2"))
            if thr > 0 and dev.nnz > 0:
                ug, vs, slots = dev.hybrid_slots(pad, thr)
                return TcLayout(ug, vs, slots, 2, "degree", regroup=thr)
            ug, vs, slots, _ = dev.hub_slots(pad, 0)
            return TcLayout(ug, vs, slots, 2, "degree")
        return super()._tc_layout(dev)

    def _onehash_rank_layout(self, dev, pad: int):
        """Edge slots for the hash-rank 1-Hash engine: the table side t of
        every edge is its higher-(degree, ID)-rank endpoint (the smaller
        largest-rank, so the other row's probes stop earliest; PG_TC_ORIENT=id:
        the lower ID), rows grouped by t and, within a row, sorted by the
        register positions the slot's probes need (pg_onehash_sort_rows), so
        the edges a warp iteration holds are equally long; row-padded to `pad`.
        Match counts are symmetric in (u, v)."""
        import ctypes
        import os
        import torch
        rows = self._rank_rows()
        if rows is None or os.environ.get("PG_ONEHASH_LAYOUT", "sorted") != "sorted":
            return None
        sg = self.sketched
        cached = getattr(sg, "_onehash_rank_layout", None)
        if cached is not None and cached[0] is dev:
            return cached[1]
        d = self._dev()
        orient = os.environ.get("PG_TC_ORIENT", "degree")
        k = sg.capacity
        group = 32 // N.onehash_block_pad(k)
        half = dev.nnz // 2
        if orient == "degree":
            # rows = in-lists of the degree orientation: row t holds its
            # lower-ranked neighbours (the probe endpoints)
            rank = dev.degree_rank()[0]
            off = torch.empty(dev.n + 1, dtype=torch.int64, device="cuda")
            adj = torch.empty(max(1, half), dtype=torch.int32, device="cuda")
            N.call("pg_degree_in_lists", N.ptr(dev.offsets), N.ptr(dev.adj), dev.n, dev.nnz,
                   N.ptr(rank), N.ptr(off), N.ptr(adj), N.stream_handle())
        else:
            ts, adj = dev.upper_edges()  # rows = u, entries = v > u
            off = torch.zeros(dev.n + 1, dtype=torch.int64, device="cuda")
            off[1:] = torch.cumsum(torch.bincount(ts, minlength=dev.n), 0)
        count = half
        ps = torch.empty(max(1, count), dtype=torch.int32, device="cuda")
        N.call("pg_onehash_sort_rows", N.ptr(off), N.ptr(adj), dev.n, N.ptr(rows), N.ptr(d["lengths"]),
               k, group, N.ptr(ps), N.stream_handle())
        del adj
        cap = count + (pad - 1) * dev.n + 1
        us = torch.empty(cap, dtype=torch.int32, device="cuda")
        vs = torch.empty(cap, dtype=torch.int32, device="cuda")
        ws_bytes = ctypes.c_size_t()
        N.call("pg_csr_upper_edges_workspace", dev.n, cap, ctypes.byref(ws_bytes))
        ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device="cuda")
        slots = ctypes.c_int64()
        N.call("pg_csr_row_slots_padded", N.ptr(off), N.ptr(ps), dev.n, pad, N.ptr(us), N.ptr(vs), cap,
               ctypes.byref(slots), N.ptr(ws), ws_bytes.value, N.stream_handle())
        torch.cuda.current_stream().synchronize()
        lay = TcLayout(us[:slots.value], vs[:slots.value], slots.value, True, orient + "+onehash-rank")
        sg._onehash_rank_layout = (dev, lay)
        return lay

    def _pairs_launch(self, us_ptr, vs_ptr, count, out_ptr):
        d, sg = self._dev(), self.sketched
        N.call("pg_pairs_minhash", N.ptr(d["entries"]), sg.capacity, int(self.onehash),
               N.ptr(d["sizes"]), us_ptr, vs_ptr, count, None, out_ptr, N.stream_handle())

    def _pairs_device(self, us, vs):
        import torch
        out = torch.empty(max(1, us.numel()), dtype=torch.float64, device="cuda")
        self._pairs_launch(N.ptr(us), N.ptr(vs), us.numel(), N.ptr(out))
        return out[:us.numel()]

    def pair_counts(self, us, vs):
        """Per-edge match counts (positional for k-Hash, set for 1-Hash)."""
        import torch
        du, on_dev = _as_device_ids(us, self.sketched.n)
        dv, _ = _as_device_ids(vs, self.sketched.n)
        d, sg = self._dev(), self.sketched
        out = torch.empty(max(1, du.numel()), dtype=torch.int32, device="cuda")
        N.call("pg_pairs_minhash", N.ptr(d["entries"]), sg.capacity,
               int(self.onehash), N.ptr(d["sizes"]), N.ptr(du), N.ptr(dv),
               du.numel(), N.ptr(out), None, N.stream_handle())
        out = out[:du.numel()]
        return out if on_dev else out.cpu().numpy().astype(np.int64)

    def _rank_rows(self):
        """1-Hash hash-rank rows for the fused pass (pg_onehash_rank_rows),
        built once per sketch; None when the engine does not take them
        (PG_ONEHASH_ROWS=id keeps the ID rows)."""
        import os
        import torch
        sg = self.sketched
        if (not self.onehash or sg.capacity not in (32, 64, 128) or sg.n == 0
                or os.environ.get("PG_ONEHASH_ROWS", "rank") != "rank"):
            return None
        d = self._dev()
        if "rank_rows" not in d:
            rank_of = torch.empty(sg.n, dtype=torch.int32, device="cuda")
            N.call("pg_hash_rank_table", sg.n, N.ptr(d["seeds"]), N.ptr(rank_of), N.stream_handle())
            rows = torch.empty_like(d["entries"])
            N.call("pg_onehash_rank_rows", N.ptr(d["entries"]), sg.n, sg.capacity, N.ptr(rank_of),
                   32 // N.onehash_block_pad(sg.capacity), N.ptr(rows), N.stream_handle())
            sg._dev["rank_rows"] = rows
            d = self._dev()
        return d["rank_rows"]

    def _tc_counts(self, us, vs, e_begin: int, e_end: int, padded: bool = False):
        import torch
        d, sg = self._dev(), self.sketched
        k = sg.capacity
        # [cnt(k+1) | ssum(k+1) | verbatim]: one buffer, one memset
        out = torch.empty(2 * k + 3, dtype=torch.int64, device="cuda")
        p0 = N.ptr(out)
        rows, mode = d["entries"], int(self.onehash)
        if self.onehash and padded:
            rr = self._rank_rows()
            if rr is not None:
                rows, mode = rr, 2
        N.call("pg_tc_minhash", N.ptr(rows), k, mode,
               N.ptr(d["sizes"]), N.ptr(us), N.ptr(vs), e_begin, e_end,
               int(padded), p0, p0 + 8 * (k + 1), p0 + 16 * (k + 1), N.stream_handle())
        return out

    def _tc_combine(self, counts: np.ndarray) -> float:
        k = self.sketched.capacity
        ssum, verb = counts[k + 1:2 * k + 2], int(counts[-1])
        terms = []
        for m in np.nonzero(ssum)[0]:
            j = float(m) / k
            terms.append((j / (1.0 + j)) * float(ssum[m]))
        return math.fsum(terms) + float(verb)

    def with_set(self, w: int, members) -> float:
        sg = self.sketched
        got = self._with_set_device(w, members, N.PG_ONEHASH if self.onehash else N.PG_KHASH,
                                    sg.capacity)
        if got is not None:
            return got
        members = np.asarray(members, dtype=np.int64)
        if sg.kind is SketchKind.KHASH:
            mem = build_khash(members, sg.capacity, sg.family)
        else:
            mem = build_onehash(members, sg.capacity, sg.family)
        return est_intersection_minhash(sg.sketch(w), mem, int(self.sizes[w]),
                                        len(members))

    def common_members(self, u: int, v: int) -> np.ndarray:
        a, b = self.sketched.sketch(u).entries, self.sketched.sketch(v).entries
        return np.intersect1d(np.unique(a), np.unique(b))


class KmvProvider(_SketchProvider):
    def __init__(self, sketched: SketchedGraph):
        sketched = as_sketched_graph(sketched)
        if sketched.kind is not SketchKind.KMV:
            raise ValueError("KmvProvider needs KMV sketches")
        super().__init__(sketched)
        self.kind = EstimatorKind.KMV

    def _pairs_launch(self, us_ptr, vs_ptr, count, out_ptr):
        d, sg = self._dev(), self.sketched
        N.call("pg_pairs_kmv", N.ptr(d["values"]), N.ptr(d["lengths"]), sg.capacity,
               N.ptr(d["sizes"]), us_ptr, vs_ptr, count, None, None, None, out_ptr,
               N.stream_handle())

    def _pairs_device(self, us, vs):
        import torch
        out = torch.empty(max(1, us.numel()), dtype=torch.float64, device="cuda")
        self._pairs_launch(N.ptr(us), N.ptr(vs), us.numel(), N.ptr(out))
        return out[:us.numel()]

    def pair_stats(self, us, vs):
        """Per-edge (common, union) counts of the stored values."""
        import torch
        du, _ = _as_device_ids(us, self.sketched.n)
        dv, _ = _as_device_ids(vs, self.sketched.n)
        d, sg = self._dev(), self.sketched
        n = max(1, du.numel())
        com = torch.empty(n, dtype=torch.int32, device="cuda")
        uni = torch.empty(n, dtype=torch.int32, device="cuda")
        N.call("pg_pairs_kmv", N.ptr(d["values"]), N.ptr(d["lengths"]),
               sg.capacity, N.ptr(d["sizes"]), N.ptr(du), N.ptr(dv), du.numel(),
               N.ptr(com), N.ptr(uni), None, None, N.stream_handle())
        return (com[:du.numel()].cpu().numpy().astype(np.int64),
                uni[:du.numel()].cpu().numpy().astype(np.int64))

    def _ranked(self) -> bool:
        """Rank rows built with the sketches (device builds) and a
        rank-directory engine for this k."""
        return "ranks" in self._dev() and N.kmv_ranked_pad(self.sketched.capacity) > 0

    def _merge_engine(self) -> bool:
        """The thread-per-edge merge engine (pg_tc_kmv_merge) over rank rows;
        PG_KMV_ENGINE=ranked restores the rank-directory engine."""
        import os
        return ("ranks" in self._dev() and N.kmv_merge_supported(self.sketched.capacity)
                and os.environ.get("PG_KMV_ENGINE", "merge") == "merge")

    def tc_pad(self) -> int:
        if self._merge_engine():
            return 1
        return N.kmv_ranked_pad(self.sketched.capacity) if self._ranked() else 1

    def _tc_layout(self, dev):
        """Merge engine: every edge once from its lower- to its higher-(degree,
        ID)-rank endpoint (so k_eff, the merge length, is the low-degree
        side's and the streamed v rows are the hub side), stably partitioned
        into [merges that stop after k_eff steps | full merges]
        (pg_kmv_merge_partition).  The estimate is symmetric in (u, v)."""
        import ctypes
        import os
        import torch
        if not self._merge_engine() or dev.n == 0:
            return super()._tc_layout(dev)
        sg = self.sketched
        cached = getattr(sg, "_kmv_merge_layout", None)
        if cached is not None and cached[0] is dev:
            return cached[1]
        d = self._dev()
        if os.environ.get("PG_TC_ORIENT", "degree") == "degree":
            us, vs, slots, _ = dev.hub_slots(1, 0)
            kind = "degree"
        else:
            us, vs = dev.upper_edges()
            slots, kind = us.numel(), "id"
        if os.environ.get("PG_KMV_PARTITION", "1") == "1" and slots > 0:
            pu, pv = torch.empty_like(us), torch.empty_like(vs)
            split = ctypes.c_int64()
            N.call("pg_kmv_merge_partition", N.ptr(us), N.ptr(vs), slots, N.ptr(d["sizes"]),
                   N.ptr(d["lengths"]), sg.capacity, int(os.environ.get("PG_KMV_BUCKETS", "8")),
                   N.ptr(pu), N.ptr(pv), ctypes.byref(split), N.stream_handle())
            us, vs = pu, pv
            split = split.value
        else:
            split = None
        lay = TcLayout(us, vs, slots, False, kind + "+kmv-merge", split=split)
        sg._kmv_merge_layout = (dev, lay)
        return lay

    def _tc_counts_shard(self, lay, rank: int, world: int):
        """Partitioned merge layout: a rank takes its balanced share of the
        k_eff-step merges and of the full merges (which run ~2x longer per
        slot and all sit at the end of the slot list), two passes."""
        if world == 1 or getattr(lay, "split", None) is None:
            return super()._tc_counts_shard(lay, rank, world)
        from .sharding import edge_range
        b0, e0 = edge_range(lay.split, rank, world)
        b1, e1 = edge_range(lay.slots - lay.split, rank, world)
        return (self._tc_counts_layout(lay, b0, e0)
                + self._tc_counts_layout(lay, lay.split + b1, lay.split + e1))

    def _tc_counts(self, us, vs, e_begin: int, e_end: int, padded: bool = False):
        import torch
        d, sg = self._dev(), self.sketched
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        if self._merge_engine():
            N.call("pg_tc_kmv_merge", N.ptr(d["ranks"]), N.ptr(d["rank_values"]),
                   N.ptr(d["lengths"]), sg.capacity, N.ptr(d["sizes"]), N.ptr(us),
                   N.ptr(vs), e_begin, e_end, N.ptr(out), N.stream_handle())
            return out
        if padded and self._ranked():
            N.call("pg_tc_kmv_ranked", N.ptr(d["ranks"]), N.ptr(d["rank_values"]),
                   N.ptr(d["lengths"]), sg.capacity, N.ptr(d["sizes"]), N.ptr(us),
                   N.ptr(vs), e_begin, e_end, N.ptr(out), N.stream_handle())
            return out
        N.call("pg_tc_kmv", N.ptr(d["values"]), N.ptr(d["lengths"]),
               sg.capacity, N.ptr(d["sizes"]), N.ptr(us), N.ptr(vs), e_begin,
               e_end, N.ptr(out), N.stream_handle())
        return out

    def _tc_combine(self, counts: np.ndarray) -> float:
        return float(counts[0])

    def with_set(self, w: int, members) -> float:
        sg = self.sketched
        got = self._with_set_device(w, members, N.PG_KMV, sg.capacity)
        if got is not None:
            return got
        members = np.asarray(members, dtype=np.int64)
        mem = build_kmv(members, sg.capacity, sg.family)
        return est_intersection_kmv(sg.sketch(w), mem, int(self.sizes[w]),
                                    len(members))


def make_provider(kind, *, graph: CsrGraph | None = None,
                  view: DirectedView | None = None,
                  sketched: SketchedGraph | None = None) -> IntersectionProvider:
    """Reference providers.py:310-338.  Graphs, views and sketches may be
    this package's objects or any objects with the reference's fields
    (adopted by value: as_csr_graph / as_directed_view / as_sketched_graph)."""
    kind = EstimatorKind(getattr(kind, "value", kind))
    if graph is not None:
        graph = as_csr_graph(graph)
    if view is not None:
        view = as_directed_view(view)
    if sketched is not None:
        sketched = as_sketched_graph(sketched)
    if kind in (EstimatorKind.EXACT_MERGE, EstimatorKind.EXACT_GALLOP):
        strategy = "gallop" if kind is EstimatorKind.EXACT_GALLOP else "merge"
        if view is not None:
            return ExactProvider.for_view(view, strategy)
        if graph is not None:
            return ExactProvider.for_graph(graph, strategy)
        raise ValueError("exact provider needs a graph or a directed view")
    if sketched is None:
        raise ValueError(f"{kind.value} provider needs sketches")
    if kind in (EstimatorKind.BF_AND, EstimatorKind.BF_L, EstimatorKind.BF_OR):
        return BloomProvider(sketched, kind)
    if kind in (EstimatorKind.KHASH, EstimatorKind.ONEHASH):
        provider = MinHashProvider(sketched)
        if provider.kind is not kind:
            raise ValueError(f"sketches are {sketched.kind.value}, "
                             f"estimator wants {kind.value}")
        return provider
    return KmvProvider(sketched)
