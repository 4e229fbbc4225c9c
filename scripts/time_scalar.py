"""Latency of the scalar API calls (pair, with_set, est_*) on device-built
sketches: mean over 200 calls after warm-up (R-MAT s20)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402

g = pg.generate_kronecker(20, 16, 1)
view = pg.degree_order(g)
e = g.edges()
rng = np.random.default_rng(0)
idx = rng.choice(len(e), 200, replace=False)
for kind, kw in (("bf_and", {"b": 2, "bits_override": 1024}), ("khash", {"k_override": 32}),
                 ("onehash", {"k_override": 32}), ("kmv", {"k_override": 32})):
    sk = pg.build_sketched_graph(g, "bloom" if kind == "bf_and" else kind, s=1.0, **kw)
    p = pg.make_provider(kind, sketched=sk)
    for i in idx[:5]:
        p.pair(int(e[i, 0]), int(e[i, 1]))
    t = time.perf_counter()
    for i in idx:
        p.pair(int(e[i, 0]), int(e[i, 1]))
    pair_us = (time.perf_counter() - t) / len(idx) * 1e6
    mem = view.adjacency[view.offsets[1000]:view.offsets[1000] + 8]
    for _ in range(5):
        p.with_set(int(e[idx[0], 0]), mem)
    t = time.perf_counter()
    for i in idx:
        p.with_set(int(e[i, 0]), mem)
    ws_us = (time.perf_counter() - t) / len(idx) * 1e6
    print(f"{kind}: pair {pair_us:.1f} us, with_set {ws_us:.1f} us", flush=True)
