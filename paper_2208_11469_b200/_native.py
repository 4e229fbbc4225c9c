"""ctypes binding of the C-ABI engine library (include/probgraph_b200.h).

The library is built in-tree (``paper_2208_11469_b200/_lib``) for sm_100a.
There is no CPU fallback: every compute entry point of this package goes
through :func:`lib`, which raises :class:`NativeUnavailable` when the shared
library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PG_LIB_PATH") or os.path.join(_HERE, "_lib", "libprobgraph_b200.so")

PG_OK = 0
PG_ERR_INVALID = -1
PG_ERR_CUDA = -2
PG_ERR_UNSUPPORTED = -3

PG_BF_AND, PG_BF_L, PG_BF_OR, PG_KHASH, PG_ONEHASH, PG_KMV = range(6)

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_dbl = ctypes.c_double
c_size = ctypes.c_size_t
c_ptr = ctypes.c_void_p

# name -> argtypes (all return int status)
SIGNATURES = {
    "pg_abi_version": [],
    "pg_last_error": [ctypes.c_char_p, c_size],
    "pg_device_sm_count": [ctypes.POINTER(ctypes.c_int)],
    "pg_family_seeds": [c_u64, c_i32, ctypes.POINTER(c_u64)],
    "pg_family_seeds_device": [c_u64, c_i32, c_ptr, c_ptr],
    "pg_hash_words": [c_ptr, c_i64, c_u64, c_ptr, c_ptr],
    "pg_csr_upper_edges_workspace": [c_i64, c_i64, ctypes.POINTER(c_size)],
    "pg_csr_upper_edges": [c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_i64,
                           ctypes.POINTER(c_i64), c_ptr, c_size, c_ptr],
    "pg_csr_upper_edges_padded": [c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr,
                                  c_i64, ctypes.POINTER(c_i64), c_ptr, c_size,
                                  c_ptr],
    "pg_group_pad": [c_i32, ctypes.POINTER(c_i32)],
    "pg_csr_row_slots_padded": [c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr,
                                c_i64, ctypes.POINTER(c_i64), c_ptr, c_size,
                                c_ptr],
    "pg_hub_tag": [c_ptr, c_i64, c_i32, c_ptr, c_i64, c_ptr, c_ptr],
    "pg_tc_bloom_hub_capacity": [c_i32, ctypes.POINTER(c_i32)],
    "pg_tc_bloom_hub": [c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_i64,
                        c_i64, c_ptr, c_i32, c_ptr, c_ptr, c_ptr],
    "pg_csr_range_slots_workspace": [c_i64, c_i64, ctypes.POINTER(c_size)],
    "pg_csr_range_slots_append": [c_ptr, c_ptr, c_i64, c_i64, c_i32, c_i32, c_i64,
                                  c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_ptr, c_size, c_ptr],
    "pg_tc_bloom_range": [c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_ptr,
                          c_i64, c_i32, c_ptr, c_ptr, c_ptr],
    "pg_csr_expand_rows": [c_ptr, c_i64, c_i64, c_ptr, c_ptr],
    "pg_build_bloom": [c_ptr, c_ptr, c_i64, c_i32, c_i32, c_ptr, c_ptr, c_ptr,
                       c_ptr],
    "pg_build_khash": [c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr],
    "pg_build_onehash": [c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr,
                         c_ptr],
    "pg_build_kmv": [c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr, c_ptr],
    "pg_kmv_rank_table": [c_i64, c_ptr, c_ptr, c_ptr, c_ptr],
    "pg_build_kmv_ranked": [c_ptr, c_ptr, c_i64, c_i32, c_ptr, c_ptr, c_ptr,
                            c_ptr, c_ptr, c_ptr, c_ptr],
    "pg_pairs_bloom": [c_ptr, c_i32, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_ptr,
                       c_i64, c_ptr, c_ptr, c_ptr],
    "pg_pairs_minhash": [c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_i64,
                         c_ptr, c_ptr, c_ptr],
    "pg_pairs_kmv": [c_ptr, c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_i64, c_ptr,
                     c_ptr, c_ptr, c_ptr, c_ptr],
    "pg_tc_bloom": [c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_i64,
                    c_i64, c_i32, c_ptr, c_ptr, c_ptr],
    "pg_tc_minhash": [c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_ptr, c_i64, c_i64,
                      c_i32, c_ptr, c_ptr, c_ptr, c_ptr],
    "pg_tc_kmv": [c_ptr, c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_i64, c_i64,
                  c_ptr, c_ptr],
    "pg_kmv_ranked_pad": [c_i32, ctypes.POINTER(c_i32)],
    "pg_onehash_block_pad": [c_i32, ctypes.POINTER(c_i32)],
    "pg_tc_kmv_ranked": [c_ptr, c_ptr, c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_i64,
                         c_i64, c_ptr, c_ptr],
    "pg_hash_rank_table": [c_i64, c_ptr, c_ptr, c_ptr],
    "pg_onehash_rank_rows": [c_ptr, c_i64, c_i32, c_ptr, c_i32, c_ptr, c_ptr],
    "pg_onehash_prefix_counts": [c_ptr, c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_i64, c_ptr, c_ptr],
    "pg_onehash_sort_rows": [c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_i32, c_i32, c_ptr, c_ptr],
    "pg_degree_in_lists": [c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr],
    "pg_kmv_merge_supported": [c_i32, ctypes.POINTER(c_i32)],
    "pg_tc_kmv_merge": [c_ptr, c_ptr, c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_i64,
                        c_i64, c_ptr, c_ptr],
    "pg_kmv_merge_partition": [c_ptr, c_ptr, c_i64, c_ptr, c_ptr, c_i32, c_i32, c_ptr, c_ptr,
                               ctypes.POINTER(c_i64), c_ptr],
    "pg_jaccard_count_khash": [c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_i64,
                               c_i64, c_i32, c_i32, c_dbl, c_ptr, c_ptr],
    "pg_4clique_bloom": [c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_i32,
                         c_i32, c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr,
                         c_ptr, c_ptr],
    "pg_4clique_bloom_edges": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_i32,
                               c_i32, c_ptr, c_i32, c_ptr, c_ptr, c_ptr, c_ptr,
                               c_ptr, c_ptr],
    "pg_4clique_exact": [c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr],
    "pg_4clique_exact_rows": [c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr,
                              c_ptr],
    "pg_4clique_sketch_workspace_size": [c_i32, c_i32, c_i64, ctypes.POINTER(c_size)],
    "pg_with_set": [c_i32, c_ptr, c_ptr, c_ptr, c_i32, c_i32, c_ptr, c_ptr, c_i32, c_ptr, c_i32,
                    c_ptr, c_ptr],
    "pg_4clique_sketch": [c_i32, c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr,
                          c_ptr, c_i32, c_ptr, c_i64, c_ptr, c_size, c_ptr, c_ptr, c_ptr],
    "pg_pairs_exact": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_ptr],
    "pg_tc_exact": [c_ptr, c_ptr, c_ptr, c_ptr, c_i64, c_ptr, c_ptr],
    "pg_two_hop_candidates": [c_ptr, c_ptr, c_i64, c_ptr, c_i64, ctypes.POINTER(c_i64),
                              c_ptr],
    "pg_similarity_scores": [c_i32, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_i32, c_ptr,
                             c_i32, c_ptr, c_ptr, c_ptr, c_ptr],
    "pg_rank_top_hits": [c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_i64, c_ptr, c_ptr],
    "pg_degree_order": [c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_ptr, c_ptr],
    "pg_jp_components": [c_ptr, c_ptr, c_ptr, c_i64, c_dbl, c_i64, c_ptr,
                         c_ptr, c_ptr],
    "pg_l2_flush": [c_ptr, c_size, c_ptr],
    "pg_rmat_pairs": [c_u64, c_u64, c_u64, c_u64, c_i32, c_i64, c_dbl, c_dbl,
                      c_dbl, c_ptr, c_ptr, c_ptr],
    "pg_pcg64_uniform": [c_u64, c_u64, c_u64, c_u64, c_i64, c_i64, c_ptr,
                         c_ptr],
    "pg_searchsorted_right": [c_ptr, c_i64, c_ptr, c_i64, c_ptr, c_ptr],
    "pg_csr_from_pairs": [c_ptr, c_ptr, c_i64, c_i64, c_ptr, c_ptr, c_i64,
                          ctypes.POINTER(c_i64), c_ptr],
}


class NativeUnavailable(RuntimeError):
    """The CUDA engine library (or a CUDA device) is not available."""


class EngineError(RuntimeError):
    """A CUDA-side failure reported by the engine."""


_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and bind every declared symbol (no GPU use)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"engine library not built: {path} (run __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = ctypes.c_int
        _lib = lib
        return lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(512)
    load_library().pg_last_error(buf, 512)
    return buf.value.decode("utf-8", "replace")


def check(rc: int, what: str = "") -> None:
    """Map a C status to the reference's exception classes."""
    if rc == PG_OK:
        return
    msg = last_error()
    if rc == PG_ERR_INVALID:
        raise ValueError(msg or what)
    if rc == PG_ERR_UNSUPPORTED:
        from .providers import UnsupportedCombinationError
        raise UnsupportedCombinationError(msg or what)
    raise EngineError(f"{what}: {msg}")


def lib():
    """The bound library, after checking that a CUDA device is usable."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable(
            "paper_2208_11469_b200 needs a CUDA device (B200, sm_100a); "
            "there is no CPU fallback")
    return load_library()


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def group_pad(row_bytes: int) -> int:
    """Lane-group size of the fused row kernels = pad of their slot layout."""
    pad = ctypes.c_int32()
    check(load_library().pg_group_pad(int(row_bytes), ctypes.byref(pad)), "pg_group_pad")
    return pad.value


def kmv_ranked_pad(k: int) -> int:
    """Slot pad of the rank-directory KMV engine for k (0: no such engine)."""
    pad = ctypes.c_int32()
    check(load_library().pg_kmv_ranked_pad(int(k), ctypes.byref(pad)), "pg_kmv_ranked_pad")
    return pad.value


def kmv_merge_supported(k: int) -> bool:
    """Whether the thread-per-edge KMV merge engine serves this k."""
    ok = ctypes.c_int32()
    check(load_library().pg_kmv_merge_supported(int(k), ctypes.byref(ok)), "pg_kmv_merge_supported")
    return bool(ok.value)


def onehash_block_pad(k: int) -> int:
    """Slot pad of the per-warp-table 1-Hash TC engine for k (1: none)."""
    pad = ctypes.c_int32()
    check(load_library().pg_onehash_block_pad(int(k), ctypes.byref(pad)), "pg_onehash_block_pad")
    return pad.value


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
