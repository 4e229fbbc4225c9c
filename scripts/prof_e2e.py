"""Phase breakdown of bench.py's e2e step (dev tool).

    python scripts/prof_e2e.py [--scale 20]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
g = pg.generate_kronecker(args.scale, 16, 1)


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


off_h = pinned(g.offsets)
adj_h = pinned(g.adjacency.astype(np.int32))
for rep in range(args.reps):
    marks = []

    def mark(name):
        torch.cuda.synchronize()
        marks.append((name, time.perf_counter()))

    mark("start")
    graph = pg.CsrGraph(off_h, adj_h)
    mark("CsrGraph")
    dev = graph.device()
    mark("H2D+device")
    skd = pg.build_sketched_graph(graph, "bloom", s=1.0, b=2, bits_override=1024)
    mark("build")
    p = pg.make_provider("bf_and", sketched=skd)
    lay = p._tc_layout(dev)
    mark("layout")
    from paper_2208_11469_b200.mining import tc_counts
    c = tc_counts(p, dev)
    mark("tc kernel")
    est = p._tc_combine(c.cpu().numpy()) / 3.0
    mark("D2H+combine")
    t0 = marks[0][1]
    print(" ".join(f"{n}={(t - pt) * 1e3:.3f}" for (n, t), (_, pt) in zip(marks[1:], marks[:-1])),
          f"total={(marks[-1][1] - t0) * 1e3:.3f}", est)
x = torch.empty(adj_h.shape, dtype=torch.int32, device="cuda")
src = torch.from_numpy(adj_h)
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    x.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
print(f"raw H2D {adj_h.nbytes / dt / 1e9:.1f} GB/s ({dt * 1e3:.3f} ms for {adj_h.nbytes} B)")

if os.environ.get("PG_TRACE"):
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            graph = pg.CsrGraph(off_h, adj_h)
            skd = pg.build_sketched_graph(graph, "bloom", s=1.0, b=2, bits_override=1024)
            est = pg.tc_estimate(graph, skd, "bf_and")
    prof.export_chrome_trace("gpurun_out/e2e_trace.json")
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
