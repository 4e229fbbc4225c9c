"""Median e2e step (host pinned CSR -> sketches -> tc_estimate), no syncs
inside the step (dev tool).   python scripts/time_e2e.py [--steps 30]"""
import argparse
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--steps", type=int, default=30)
args = ap.parse_args()
g = pg.generate_kronecker(args.scale, 16, 1)


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


off_h = pinned(g.offsets)
adj_h = pinned(g.adjacency.astype(np.int32))
times = []
for i in range(args.steps + 3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    graph = pg.CsrGraph(off_h, adj_h)
    sk = pg.build_sketched_graph(graph, "bloom", s=1.0, b=2, bits_override=1024)
    est = pg.tc_estimate(graph, sk, "bf_and")
    torch.cuda.synchronize()
    if i >= 3:
        times.append(time.perf_counter() - t0)
print(f"chunks={os.environ.get('PG_UPLOAD_CHUNKS', 'default')} median={statistics.median(times) * 1e3:.3f} ms "
      f"min={min(times) * 1e3:.3f} p90={sorted(times)[int(0.9 * len(times))] * 1e3:.3f} est={est}")

if os.environ.get("PG_TRACE"):
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            torch.cuda.synchronize()
            graph = pg.CsrGraph(off_h, adj_h)
            sk = pg.build_sketched_graph(graph, "bloom", s=1.0, b=2, bits_override=1024)
            est = pg.tc_estimate(graph, sk, "bf_and")
            torch.cuda.synchronize()
    prof.export_chrome_trace("gpurun_out/e2e_trace2.json")
