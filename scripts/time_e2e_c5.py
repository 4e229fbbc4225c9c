"""c5 end-to-end breakdown: raw pinned H2D of the CSR vs the public-API path
(CsrGraph(host CSR) -> build_sketched_graph -> tc_estimate), wall clock
with a device sync on both sides, median of 5."""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.environ.get("PG_REPO", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2208_11469_b200 as pg  # noqa: E402

sc = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = pg.generate_kronecker(sc, 16, 4 if sc == 24 else 1)
bits = 2048 if sc == 24 else 1024


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t


off_t, adj_t = pinned(g.offsets), pinned(g.adjacency.astype(np.int32))
off_h, adj_h = off_t.numpy(), adj_t.numpy()
nbytes = off_h.nbytes + adj_h.nbytes


def wall(fn, reps=5):
    ts = []
    for i in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        if i:
            ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


dst_o = torch.empty_like(off_t, device="cuda")
dst_a = torch.empty_like(adj_t, device="cuda")
ms_copy = wall(lambda: (dst_o.copy_(off_t, non_blocking=True), dst_a.copy_(adj_t, non_blocking=True)))
print(f"raw H2D {nbytes / 1e9:.2f} GB: {ms_copy:.2f} ms = {nbytes / ms_copy / 1e6:.1f} GB/s", flush=True)


def build_only():
    gr = pg.CsrGraph(off_h, adj_h)
    pg.build_sketched_graph(gr, "bloom", s=1.0, b=2, bits_override=bits)


def e2e():
    gr = pg.CsrGraph(off_h, adj_h)
    sk = pg.build_sketched_graph(gr, "bloom", s=1.0, b=2, bits_override=bits)
    return pg.tc_estimate(gr, sk, "bf_and")


print(f"CsrGraph + build: {wall(build_only):.2f} ms", flush=True)
print(f"e2e: {wall(e2e):.2f} ms", flush=True)

gr = pg.CsrGraph(off_h, adj_h)
sk = pg.build_sketched_graph(gr, "bloom", s=1.0, b=2, bits_override=bits)
dev = gr.device()
p = pg.make_provider("bf_and", sketched=sk)
from paper_2208_11469_b200.mining import _chunk_pipelined  # noqa: E402
print("upload chunks", len(dev.upload_chunks), "chunk_ready", len(sk._chunk_ready or []),
      "pipelined", _chunk_pipelined(p, dev), "pad", p.tc_pad(), "layouts", list(dev._layouts))
