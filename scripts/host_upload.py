"""Timers inside the chunked upload (dev tool)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200.graphs import side_stream  # noqa: E402

g = pg.generate_kronecker(20, 16, 1)


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


offsets = pinned(g.offsets)
adjacency = pinned(g.adjacency.astype(np.int32))
n, nnz = len(offsets) - 1, len(adjacency)
keep = []
for rep in range(5):
    torch.cuda.synchronize()
    T = []
    t = time.perf_counter()

    def mark(name):
        global t
        now = time.perf_counter()
        T.append(f"{name}={(now - t) * 1e3:.3f}")
        t = now

    adj_t = torch.from_numpy(np.ascontiguousarray(adjacency))
    pinned_ok = adj_t.is_pinned()
    mark("from_numpy+is_pinned")
    cur = torch.cuda.current_stream()
    cs = side_stream("copy")
    o_d = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    a_d = torch.empty(nnz, dtype=torch.int32, device="cuda")
    mark("empty")
    off_t = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64))
    cuts = np.searchsorted(offsets, np.linspace(0, nnz, 9), side="left")
    cuts[0], cuts[-1] = 0, n
    cuts = np.unique(cuts)
    mark("cuts")
    cs.wait_stream(cur)
    with torch.cuda.stream(cs):
        o_d.copy_(off_t, non_blocking=True)
        mark("off copy")
        for v0, v1 in zip(cuts[:-1].tolist(), cuts[1:].tolist()):
            a, b = int(offsets[v0]), int(offsets[v1])
            a_d[a:b].copy_(adj_t[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        mark("chunks")
    o_d.record_stream(cs)
    a_d.record_stream(cs)
    cur.wait_stream(cs)
    mark("tail")
    keep.append((o_d, a_d))
    if len(keep) > 2:
        keep.pop(0)
    print(pinned_ok, " ".join(T))
