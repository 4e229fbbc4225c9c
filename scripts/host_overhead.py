"""Host-side (enqueue) cost of the e2e pieces, no syncs (dev tool)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200 import _native as N  # noqa: E402

g = pg.generate_kronecker(20, 16, 1)


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


off_h = pinned(g.offsets)
adj_h = pinned(g.adjacency.astype(np.int32))
for rep in range(4):
    torch.cuda.synchronize()
    T = {}
    t = time.perf_counter()
    graph = pg.CsrGraph(off_h, adj_h)
    T["csr"] = time.perf_counter() - t
    t = time.perf_counter()
    dev = graph.device()
    T["device"] = time.perf_counter() - t
    t = time.perf_counter()
    sk = pg.build_sketched_graph(graph, "bloom", s=1.0, b=2, bits_override=1024)
    T["build"] = time.perf_counter() - t
    p = pg.make_provider("bf_and", sketched=sk)
    from paper_2208_11469_b200.mining import tc_counts
    t = time.perf_counter()
    c = tc_counts(p, dev)
    T["tc enqueue"] = time.perf_counter() - t
    t = time.perf_counter()
    h = c.cpu().numpy()
    T["d2h"] = time.perf_counter() - t
    t = time.perf_counter()
    est = p._tc_combine(h) / 3.0
    T["combine"] = time.perf_counter() - t
    print(" ".join(f"{k}={v * 1e3:.3f}" for k, v in T.items()))
# micro: per-call costs
x = torch.empty(1 << 20, dtype=torch.int32, device="cuda")
src = torch.from_numpy(adj_h[:1 << 20])
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(100):
    x.copy_(src, non_blocking=True)
print(f"copy_ enqueue {(time.perf_counter() - t) * 1e4:.1f} us/call")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(100):
    torch.from_numpy(adj_h).is_pinned()
print(f"is_pinned {(time.perf_counter() - t) * 1e4:.1f} us/call")
seeds = torch.empty(2, dtype=torch.int64, device="cuda")
rows = torch.empty((1 << 14, 16), dtype=torch.int64, device="cuda")
ones = torch.empty(1 << 14, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(100):
    N.call("pg_build_bloom", N.ptr(dev.offsets), N.ptr(dev.adj), 1 << 14, 1024, 2, N.ptr(seeds),
           N.ptr(rows), N.ptr(ones), N.stream_handle())
print(f"pg_build_bloom enqueue {(time.perf_counter() - t) * 1e4:.1f} us/call")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(100):
    e = torch.cuda.Event()
    e.record()
print(f"event create+record {(time.perf_counter() - t) * 1e4:.1f} us/call")
