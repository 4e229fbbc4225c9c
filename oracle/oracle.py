"""CPU oracle for the per-edge sketch-intersection path.

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package (paper_2208_11469_b200), which has no CPU path.

Two restatements of the reference algorithm
(/root/reference/pkg/src/probgraph, numpy only, no third-party arithmetic):

* ``C``  -- ctypes binding of ``pg_oracle.c`` (OpenMP), used as the fast
  checker for large parity cases;
* ``NumpyPort`` -- the reference's own vectorised strategy re-stated with
  numpy (gather rows -> bitwise op -> bitwise_count -> estimate; per
  16,384-edge chunk; ThreadPoolExecutor over a fixed chunk grid, partials
  summed in chunk order; sketches.py:314-396, providers.py:137-301,
  mining.py:63-80,105-130).  This is what bench.py times as the reference
  CPU arm.

Both are pinned against fixtures produced by running the reference itself
(tests/golden/make_golden.py; tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libpgoracle.so")

M64 = (1 << 64) - 1
DEFAULT_HASH_SEED = 0x9E3779B97F4A7C15
CHUNK = 16384  # mining.py:46


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


class _C:
    _lib = None

    def lib(self):
        if self._lib is None:
            if not os.path.exists(LIB):
                build()
            L = ctypes.CDLL(LIB)
            P = ctypes.c_void_p
            i64, i32, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_uint64
            sig = {
                "pgo_family_seeds": [u64, i32, P],
                "pgo_build_bloom": [i64, P, P, i32, i32, P, P, P],
                "pgo_build_khash": [i64, P, P, i32, P, P],
                "pgo_build_onehash": [i64, P, P, i32, u64, P, P],
                "pgo_build_kmv": [i64, P, P, i32, u64, P, P],
                "pgo_pairs_bloom": [P, i32, i32, P, P, i64, P],
                "pgo_pairs_minhash": [P, i32, i32, P, P, i64, P],
                "pgo_pairs_kmv": [P, P, i32, P, P, P, i64, P, P, P],
                "pgo_pairs_exact": [P, P, P, P, i64, P],
                "pgo_4clique_bloom": [i64, P, P, P, i32, i32, P, i32, P, i64, P, P],
                "pgo_rmat_pairs": [i32, i64, u64, u64, u64, u64, P, P],
                "pgo_csr_from_pairs": [i64, i64, P, P, P, P],
                "pgo_num_threads": [],
                "pgo_set_threads": [i32],
            }
            for name, args in sig.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = {"pgo_num_threads": ctypes.c_int,
                             "pgo_csr_from_pairs": ctypes.c_int64}.get(name)
            self._lib = L
        return self._lib

    @staticmethod
    def _p(a):
        return a.ctypes.data_as(ctypes.c_void_p)

    def seeds(self, base: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        self.lib().pgo_family_seeds(base & M64, count, self._p(out))
        return out

    def generate_kronecker(self, scale: int, edge_factor: int, seed: int):
        """(offsets int64[n+1], adjacency int64[2m]) of the reference's
        generate_kronecker(scale, edge_factor, seed) (graphs.py:251-276):
        the same PCG64 draws (pgo_rmat_pairs) and CsrGraph.from_edges
        (graphs.py:57-89, pgo_csr_from_pairs), in C with OpenMP."""
        if scale < 1:
            raise ValueError("scale must be >= 1")
        n = 1 << scale
        count = edge_factor * n
        st = np.random.default_rng(seed).bit_generator.state["state"]
        src = np.empty(max(1, count), dtype=np.int32)
        dst = np.empty(max(1, count), dtype=np.int32)
        self.lib().pgo_rmat_pairs(scale, count, st["state"] >> 64, st["state"] & M64,
                                  st["inc"] >> 64, st["inc"] & M64, self._p(src), self._p(dst))
        off = np.empty(n + 1, dtype=np.int64)
        adj = np.empty(max(1, 2 * count), dtype=np.int64)
        nnz = self.lib().pgo_csr_from_pairs(n, count, self._p(src), self._p(dst),
                                            self._p(off), self._p(adj))
        del src, dst
        return off, adj[:nnz].copy()

    def set_threads(self, t: int):
        self.lib().pgo_set_threads(t)

    def num_threads(self) -> int:
        return self.lib().pgo_num_threads()

    def build_bloom(self, off, adj, bits, b, seed=DEFAULT_HASH_SEED):
        off, adj = _i64(off), _i64(adj)
        n = len(off) - 1
        s = self.seeds(seed, b)
        rows = np.empty((n, bits // 64), dtype=np.uint64)
        ones = np.empty(n, dtype=np.int64)
        self.lib().pgo_build_bloom(n, self._p(off), self._p(adj), bits, b,
                                   self._p(s), self._p(rows), self._p(ones))
        return rows, ones

    def build_khash(self, off, adj, k, seed=DEFAULT_HASH_SEED):
        off, adj = _i64(off), _i64(adj)
        n = len(off) - 1
        s = self.seeds(seed, k)
        ent = np.empty((n, k), dtype=np.int64)
        self.lib().pgo_build_khash(n, self._p(off), self._p(adj), k, self._p(s),
                                   self._p(ent))
        return ent

    def build_onehash(self, off, adj, k, seed=DEFAULT_HASH_SEED):
        off, adj = _i64(off), _i64(adj)
        n = len(off) - 1
        s0 = int(self.seeds(seed, 1)[0])
        ent = np.empty((n, k), dtype=np.int64)
        ln = np.empty(n, dtype=np.int64)
        self.lib().pgo_build_onehash(n, self._p(off), self._p(adj), k, s0,
                                     self._p(ent), self._p(ln))
        return ent, ln

    def build_kmv(self, off, adj, k, seed=DEFAULT_HASH_SEED):
        off, adj = _i64(off), _i64(adj)
        n = len(off) - 1
        s0 = int(self.seeds(seed, 1)[0])
        val = np.empty((n, k), dtype=np.float64)
        ln = np.empty(n, dtype=np.int64)
        self.lib().pgo_build_kmv(n, self._p(off), self._p(adj), k, s0,
                                 self._p(val), self._p(ln))
        return val, ln

    def pairs_bloom(self, rows, bits, use_or, us, vs):
        us, vs = _i64(us), _i64(vs)
        out = np.empty(len(us), dtype=np.int64)
        self.lib().pgo_pairs_bloom(self._p(np.ascontiguousarray(rows)), bits,
                                   2 if use_or else 0, self._p(us), self._p(vs),
                                   len(us), self._p(out))
        return out

    def pairs_minhash(self, ent, k, onehash, us, vs):
        us, vs = _i64(us), _i64(vs)
        out = np.empty(len(us), dtype=np.int64)
        self.lib().pgo_pairs_minhash(self._p(_i64(ent)), k, int(onehash),
                                     self._p(us), self._p(vs), len(us), self._p(out))
        return out

    def pairs_kmv(self, vals, lengths, k, sizes, us, vs):
        us, vs = _i64(us), _i64(vs)
        com = np.empty(len(us), dtype=np.int64)
        uni = np.empty(len(us), dtype=np.int64)
        est = np.empty(len(us), dtype=np.float64)
        self.lib().pgo_pairs_kmv(self._p(np.ascontiguousarray(vals, dtype=np.float64)),
                                 self._p(_i64(lengths)), k, self._p(_i64(sizes)),
                                 self._p(us), self._p(vs), len(us), self._p(com),
                                 self._p(uni), self._p(est))
        return com, uni, est

    def pairs_exact(self, off, adj, us, vs):
        us, vs = _i64(us), _i64(vs)
        out = np.empty(len(us), dtype=np.int64)
        self.lib().pgo_pairs_exact(self._p(_i64(off)), self._p(_i64(adj)),
                                   self._p(us), self._p(vs), len(us), self._p(out))
        return out

    def four_clique_bloom(self, off, adj, rows, bits, b, seed=DEFAULT_HASH_SEED,
                          use_or=False, edge_ids=None):
        off, adj = _i64(off), _i64(adj)
        n = len(off) - 1
        s = self.seeds(seed, b)
        hist = np.zeros(bits + 1, dtype=np.int64)
        trip = np.zeros(1, dtype=np.int64)
        ids = None if edge_ids is None else _i64(edge_ids)
        self.lib().pgo_4clique_bloom(n, self._p(off), self._p(adj),
                                     self._p(np.ascontiguousarray(rows)), bits, b,
                                     self._p(s), 2 if use_or else 0,
                                     None if ids is None else self._p(ids),
                                     0 if ids is None else len(ids),
                                     self._p(hist), self._p(trip))
        return hist, int(trip[0])


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


C = _C()


# ---------------------------------------------------------------------------
# estimate math shared by both restatements (estimators.py:65-70,
# providers.py:137-145, :223-230)


def swamidass(bits: int, b: int, ones):
    o = np.asarray(ones, dtype=np.float64)
    return -(bits / b) * np.log1p(-(o - (o == bits)) / bits)


def upper_edges(off, adj):
    """(us, vs) with u < v in CSR order (graphs.py:101-105)."""
    off, adj = _i64(off), _i64(adj)
    src = np.repeat(np.arange(len(off) - 1, dtype=np.int64), np.diff(off))
    keep = src < adj
    return src[keep], adj[keep]


def bloom_edge_estimates(pop, kind, bits, b, su=None, sv=None):
    if kind == "bf_and":
        return swamidass(bits, b, pop)
    if kind == "bf_l":
        return pop.astype(np.float64) / b
    raw = su + sv - swamidass(bits, b, pop)
    return np.maximum(raw, 0.0)


def minhash_edge_estimates(m, k, su, sv, onehash):
    m = m.astype(np.float64)
    j = m / k
    est = (j / (1.0 + j)) * (su.astype(np.float64) + sv.astype(np.float64))
    if onehash:
        est = np.where((su <= k) & (sv <= k), m, est)
    return est


# ---------------------------------------------------------------------------
# numpy port of the reference CPU path (the timed "reference" arm)


class NumpyPort:
    """The reference's vectorised CPU strategy, restated with numpy."""

    def __init__(self, threads: int | None = None):
        self.threads = threads or len(os.sched_getaffinity(0))

    # -- builders (sketches.py:314-396)
    @staticmethod
    def _hash(seed: int, keys):
        x = np.uint64(seed) ^ keys.astype(np.uint64)
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xFF51AFD7ED558CCD)
        x ^= x >> np.uint64(33)
        x *= np.uint64(0xC4CEB9FE1A85EC53)
        x ^= x >> np.uint64(33)
        return x

    def build_bloom(self, off, adj, bits, b, seed=DEFAULT_HASH_SEED):
        off, adj = _i64(off), _i64(adj)
        n = len(off) - 1
        words = bits // 64
        rows = np.zeros(n * words, dtype=np.uint64)
        owner = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
        for s in C.seeds(seed, b):
            pos = (self._hash(int(s), adj) % np.uint64(bits)).astype(np.int64)
            np.bitwise_or.at(rows, owner * words + (pos >> 6),
                             np.uint64(1) << (pos & 63).astype(np.uint64))
        rows = rows.reshape(n, words)
        return rows, np.bitwise_count(rows).sum(axis=1).astype(np.int64)

    # -- per-edge batch kernels (providers.py:150-162, 205-232, 266-301)
    @staticmethod
    def bloom_chunk(rows, bits, b, kind, sizes, us, vs):
        op = np.bitwise_or if kind == "bf_or" else np.bitwise_and
        pop = np.bitwise_count(op(rows[us], rows[vs])).sum(axis=1)
        return bloom_edge_estimates(pop, kind, bits, b,
                                    sizes[us] if kind == "bf_or" else None,
                                    sizes[vs] if kind == "bf_or" else None)

    @staticmethod
    def khash_chunk(ent, k, sizes, us, vs):
        a, c = ent[us], ent[vs]
        m = np.count_nonzero((a == c) & (a >= 0), axis=1)
        return minhash_edge_estimates(m, k, sizes[us], sizes[vs], False)

    @staticmethod
    def onehash_chunk(ent, k, sizes, us, vs):
        step = max(64, min(CHUNK, 2 ** 24 // max(1, k * k)))
        out = np.empty(len(us), dtype=np.float64)
        for lo in range(0, len(us), step):
            hi = min(lo + step, len(us))
            a, c = ent[us[lo:hi]], ent[vs[lo:hi]].copy()
            c[c < 0] = -2
            m = (a[:, :, None] == c[:, None, :]).any(axis=2).sum(axis=1)
            out[lo:hi] = minhash_edge_estimates(m, k, sizes[us[lo:hi]],
                                                sizes[vs[lo:hi]], True)
        return out

    @staticmethod
    def kmv_chunk(vals, lengths, k, sizes, us, vs):
        merged = np.sort(np.concatenate([vals[us], vals[vs]], axis=1), axis=1)
        fin = np.isfinite(merged)
        dup = (merged[:, 1:] == merged[:, :-1]) & fin[:, 1:]
        common = dup.sum(axis=1).astype(np.float64)
        first = fin.copy()
        first[:, 1:] &= ~dup
        union = first.sum(axis=1).astype(np.float64)
        su, sv = sizes[us].astype(np.float64), sizes[vs].astype(np.float64)
        keff = np.minimum(lengths[us], lengths[vs])
        pos = np.argmax(np.cumsum(first, axis=1) >= np.maximum(keff, 1)[:, None], axis=1)
        kth = merged[np.arange(len(us)), pos]
        with np.errstate(divide="ignore", invalid="ignore"):
            est_union = (keff - 1) / kth
        verbatim = (su <= k) & (sv <= k)
        raw = np.where(verbatim, su + sv - union,
                       np.where(keff < 2, common, su + sv - est_union))
        return np.clip(raw, 0.0, np.minimum(su, sv))

    # -- tc_estimate (mining.py:63-80, 105-130)
    def tc_sum(self, chunk_fn, us, vs):
        """Sum chunk_fn over the fixed 16,384-edge grid, in chunk order."""
        grid = [(lo, min(lo + CHUNK, len(us))) for lo in range(0, len(us), CHUNK)]
        if not grid:
            return 0.0

        def work(r):
            return float(chunk_fn(us[r[0]:r[1]], vs[r[0]:r[1]]).sum())

        if self.threads <= 1 or len(grid) == 1:
            parts = [work(r) for r in grid]
        else:
            with ThreadPoolExecutor(max_workers=self.threads) as pool:
                parts = list(pool.map(work, grid))
        total = parts[0]
        for p in parts[1:]:
            total = total + p
        return total
