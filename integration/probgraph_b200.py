"""Optional B200 backend for probgraph's Bloom path -- the module a maintainer
of the reference package adds as ``probgraph/b200.py``.

A ctypes binding of the C ABI in include/probgraph_b200.h; torch only owns
device memory and supplies the stream handle.  ``tc_estimate_b200`` is the
drop-in for ``mining.tc_estimate`` (reference src/mining.py:105-130) on Bloom
sketches (AND / L / OR).  tests/test_gpu_plugin_boundary.py loads this very
file as ``probgraph.b200`` inside a stand-in ``probgraph`` package and checks
it against values the reference computed.
"""
import ctypes
import math
import os

import numpy as np
import torch  # device memory + stream handle only

from .estimators import EstimatorKind, swamidass_value

_lib = ctypes.CDLL(os.environ.get("PROBGRAPH_B200_LIB", "libprobgraph_b200.so"))
P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_lib.pg_csr_upper_edges_workspace.argtypes = [I64, I64, ctypes.POINTER(ctypes.c_size_t)]
_lib.pg_csr_upper_edges.argtypes = [P, P, I64, P, P, I64, ctypes.POINTER(I64), P,
                                    ctypes.c_size_t, P]
_lib.pg_tc_bloom.argtypes = [P, I32, I32, P, P, P, P, I64, I64, I32, P, P, P]
_lib.pg_last_error.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
_OPS = {"bf_and": 0, "bf_l": 1, "bf_or": 2}


def _check(rc):
    if rc:
        buf = ctypes.create_string_buffer(512)
        _lib.pg_last_error(buf, 512)
        raise (ValueError if rc == -1 else RuntimeError)(buf.value.decode())


def tc_estimate_b200(graph, sketched, kind=EstimatorKind.BF_AND):
    """Drop-in for mining.tc_estimate on Bloom sketches (AND / L / OR)."""
    kind = EstimatorKind(kind)
    if kind.value not in _OPS:
        raise ValueError(f"{kind} is not a Bloom estimator")
    stream = torch.cuda.current_stream().cuda_stream
    off = torch.from_numpy(np.ascontiguousarray(graph.offsets, dtype=np.int64)).cuda()
    adj = torch.from_numpy(np.ascontiguousarray(graph.adjacency, dtype=np.int32)).cuda()
    rows = torch.from_numpy(np.ascontiguousarray(sketched.bit_matrix).view(np.int64)).cuda()
    sizes = torch.from_numpy(np.asarray(sketched.sizes, dtype=np.int32)).cuda()
    B, b = sketched.bit_length, sketched.hash_count
    lut_host = np.ascontiguousarray(swamidass_value(B, b, np.arange(B + 1, dtype=np.float64)),
                                    dtype=np.float64)
    lut = torch.from_numpy(lut_host).cuda()
    m = max(1, graph.m)
    us = torch.empty(m, dtype=torch.int32, device="cuda")
    vs = torch.empty(m, dtype=torch.int32, device="cuda")
    wsb = ctypes.c_size_t()
    _check(_lib.pg_csr_upper_edges_workspace(graph.n, m, ctypes.byref(wsb)))
    ws = torch.empty(max(1, wsb.value), dtype=torch.uint8, device="cuda")
    got = I64()
    _check(_lib.pg_csr_upper_edges(off.data_ptr(), adj.data_ptr(), graph.n,
                                   us.data_ptr(), vs.data_ptr(), m, ctypes.byref(got),
                                   ws.data_ptr(), wsb.value, stream))
    hist = torch.empty(B + 2, dtype=torch.int64, device="cuda")
    _check(_lib.pg_tc_bloom(rows.data_ptr(), B, _OPS[kind.value], sizes.data_ptr(),
                            lut.data_ptr(), us.data_ptr(), vs.data_ptr(), 0, got.value, 0,
                            hist.data_ptr(), hist.data_ptr() + 8 * (B + 1), stream))
    h = hist.cpu().numpy()
    h, spos = h[:-1], int(h[-1])
    if kind.value == "bf_l":
        total = float(int(np.dot(h, np.arange(B + 1)))) / b
    else:
        weighted = math.fsum(float(h[o]) * float(lut_host[o]) for o in np.nonzero(h)[0])
        total = weighted if kind.value == "bf_and" else float(spos) - weighted
    return total / 3.0
