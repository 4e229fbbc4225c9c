"""c5 Bloom TC: hub-cached degree-oriented engine vs the ID-oriented one
(CUDA-event medians, L2 flushed), hub coverage of the edge set, and the
histogram equality check.  python scripts/probe_hub.py [scale]"""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200 import _native as N  # noqa: E402
from paper_2208_11469_b200.providers import TcLayout  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
seed = {20: 1, 22: 2, 24: 4}.get(scale, 4)
g = pg.generate_kronecker(scale, 16, seed)
sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048)
p = pg.make_provider("bf_and", sketched=sk)
dev = g.device()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def tm(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        N.call("pg_l2_flush", N.ptr(flush), flush.numel(), N.stream_handle())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out


os.environ["PG_TC_HUB"] = "0"
lay0 = p._tc_layout(dev)
ms0, h0 = tm(lambda: p._tc_counts_layout(lay0, 0, lay0.slots))
print(f"id-oriented: {ms0:.3f} ms slots={lay0.slots} m={g.m}", flush=True)
os.environ["PG_TC_HUB"] = "1"
cap = p.hub_capacity()
rank, off, adj = dev.degree_rank()
indeg = torch.bincount(adj.long(), minlength=g.n)
order = torch.argsort(rank.long(), descending=True)
cum = torch.cumsum(indeg[order], 0).cpu().numpy()
for H in (cap // 2, cap, 2 * cap, 8 * cap, 100000):
    print(f"coverage H={H}: {cum[H - 1] / g.m:.4f}")
od = (off[1:] - off[:-1]).cpu().numpy()
print("N+ runs mean", od[od > 0].mean(), "pad8 slots/m", (np.ceil(od / 8) * 8).sum() / g.m)
for hubs in (0, cap // 2, cap):
    ug, vs, slots, hid = dev.hub_slots(8, hubs)
    lay = TcLayout(ug, vs, slots, 2, "hub", hid, hubs)
    ms, h = tm(lambda: p._tc_counts_layout(lay, 0, slots))
    same = torch.equal(h, h0)
    print(f"hub H={hubs} threads={os.environ.get('PG_HUB_THREADS', 768)} csa={os.environ.get('PG_HUB_CSA', 1)}: {ms:.3f} ms slots={slots} same={same}", flush=True)
