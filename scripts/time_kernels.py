"""Median CUDA-event time of one estimator pass per config, L2 flushed before
each timed call (outside the events).

    python scripts/time_kernels.py c4 | c5 | c3onehash | c3kmv | c5b_khash | c5b_onehash | c5b_kmv | c5b_bloom
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200 import _native as N  # noqa: E402
from paper_2208_11469_b200.mining import (four_clique_counts, four_clique_sketch_sum,  # noqa: E402
                                          jaccard_counts, tc_counts)

flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=7):
    st = torch.cuda.current_stream()
    fn()
    fn()
    ts = []
    for _ in range(reps):
        N.call("pg_l2_flush", N.ptr(flush_buf), flush_buf.numel(), N.stream_handle())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        out = fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out


for cfg in sys.argv[1:]:
    if cfg == "c4":
        g = pg.generate_chung_lu(1 << 23, 32, 2.1, 3)
        sk = pg.build_sketched_graph(g, "khash", s=1.0, k_override=32)
        ms, out = timeit(lambda: jaccard_counts(g, sk, 0.1))
        print(cfg, os.environ.get("PG_TC_ORIENT", ""), f"{ms:.3f} ms", out[:2].tolist(), flush=True)
    elif cfg in ("c5", "c2"):
        sc, seed, bits = (24, 4, 2048) if cfg == "c5" else (20, 1, 1024)
        g = pg.generate_kronecker(sc, 16, seed)
        sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=bits)
        p = pg.make_provider("bf_and", sketched=sk)
        dev = g.device()
        ms, out = timeit(lambda: tc_counts(p, dev))
        print(cfg, f"{ms:.3f} ms", p._tc_combine(out.cpu().numpy()) / 3.0, flush=True)
    elif cfg in ("c3onehash", "c3kmv"):
        g = pg.generate_kronecker(22, 16, 2)
        kind = cfg[2:]
        sk = pg.build_sketched_graph(g, kind, s=1.0, k_override=64)
        p = pg.make_provider(kind, sketched=sk)
        ms, out = timeit(lambda: tc_counts(p, g.device()))
        print(cfg, f"{ms:.3f} ms", p._tc_combine(out.cpu().numpy()) / 3.0, flush=True)
    elif cfg.startswith("c5b_"):
        kind = cfg[4:]
        g = pg.generate_kronecker(18, 16, 4)
        view = pg.degree_order(g)
        if kind == "bloom":
            dsk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048,
                                          source="directed", view=view)
            p = pg.make_provider("bf_and", sketched=dsk)
            nnz = view.device().nnz
            ms, out = timeit(lambda: four_clique_counts(view, p, 0, nnz), reps=3)
            print(cfg, f"{ms:.3f} ms", int(out[-1]), flush=True)
        else:
            k = int(os.environ.get("PG_K", "64"))
            dsk = pg.build_sketched_graph(g, kind, s=1.0, k_override=k, source="directed", view=view)
            p = pg.make_provider(kind, sketched=dsk)
            ms, out = timeit(lambda: four_clique_sketch_sum(view, p), reps=3)
            print(cfg, k, f"{ms:.3f} ms", out, f"{out[1] / ms / 1e6:.2f} G triples/s", flush=True)
