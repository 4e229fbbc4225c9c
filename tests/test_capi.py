"""The C-ABI library loads and exports exactly what include/*.h declares.

No compute calls here: this runs without a GPU.
"""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "probgraph_b200.h")
LIB = os.path.join(REPO, "paper_2208_11469_b200", "_lib", "libprobgraph_b200.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"PG_API\s+int\s+(pg_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("pg_build_bloom", "pg_build_khash", "pg_build_onehash", "pg_build_kmv",
                 "pg_pairs_bloom", "pg_pairs_minhash", "pg_pairs_kmv", "pg_tc_bloom",
                 "pg_tc_minhash", "pg_tc_kmv", "pg_jaccard_count_khash",
                 "pg_4clique_bloom", "pg_family_seeds", "pg_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(pg_\w+)", out))
    assert set(declared()) <= exported
    # nothing beyond the ABI leaks out of the library
    assert {s for s in exported if s.startswith("pg_")} == set(declared())


def test_binding_covers_header_and_loads():
    from paper_2208_11469_b200 import _native as N
    assert set(N.SIGNATURES) == set(declared())
    lib = N.load_library()
    assert lib.pg_abi_version() == 1


def test_seed_derivation_and_error_reporting_without_gpu():
    from paper_2208_11469_b200 import _native as N
    lib = N.load_library()
    out = (ctypes.c_uint64 * 2)()
    assert lib.pg_family_seeds(0x9E3779B97F4A7C15, 2, out) == 0
    assert (out[0], out[1]) == (0x2D0A2CC335CD72A7, 0x95527B2E69B24CDF)
    assert lib.pg_family_seeds(1, 0, out) == N.PG_ERR_INVALID
    assert "at least one" in N.last_error()
    # argument validation happens before any device work
    rc = lib.pg_build_bloom(None, None, 10, 100, 1, None, None, None, None)
    assert rc == N.PG_ERR_INVALID
    assert "multiple of 64" in N.last_error()
    # k > 256 has a generic device path: only the null pointers are rejected
    rc = lib.pg_build_khash(None, None, 10, 1000, None, None, None)
    assert rc == N.PG_ERR_INVALID
    assert "null pointer" in N.last_error()
    # an engine-specific range is reported as unsupported (callers fall back)
    rc = lib.pg_tc_kmv_ranked(None, None, None, 40, None, None, None, 0, 1, None, None)
    assert rc == N.PG_ERR_UNSUPPORTED
    with pytest.raises(ValueError):
        N.check(N.PG_ERR_INVALID)


def test_product_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200._native import NativeUnavailable
    g = pg.CsrGraph.from_edges([(0, 1), (1, 2), (2, 0)])
    with pytest.raises((NativeUnavailable, RuntimeError, AssertionError)):
        pg.build_sketched_graph(g, "bloom", s=1.0, bits_override=64)


def test_sm100a_code_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
