"""Probe what bounds the Bloom TC kernel: time it on crafted edge lists.

A real  : the c2 upper edge list (CSR order)
B l2res : real u, v replaced by a random vertex < 65536 (rows L2-resident)
C same  : v = u (second row is an L1 hit)
D shuffled: the real edges in random order (no u-row reuse)
Also a torch clone of a 32 MiB buffer (L2-resident copy) and of 1 GiB (HBM).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200 import _native as N  # noqa: E402

bits = int(os.environ.get("BITS", "1024"))
cache = "/tmp/pg_rmat_20_16_1.npz"
if os.path.exists(cache):
    z = np.load(cache)
    g = pg.CsrGraph(z["o"], z["a"])
else:
    g = pg.generate_kronecker(20, 16, 1)
    np.savez(cache, o=g.offsets, a=g.adjacency)
sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=bits)
p = pg.make_provider("bf_and", sketched=sk)
us, vs = g.device().upper_edges()
m = us.numel()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()


def timeit(u, v, reps=10):
    ts = []
    for i in range(reps + 2):
        N.call("pg_l2_flush", N.ptr(flush), flush.numel(), N.stream_handle())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        p._tc_counts(u, v, 0, u.numel())
        b.record(st)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts))


gen = torch.Generator(device="cuda").manual_seed(0)
res = {"bits": bits, "engine": os.environ.get("PG_TC_ENGINE", "staged"),
       "vcache": "PG_TC_VCACHE" in os.environ}
res["A_real"] = timeit(us, vs)
res["B_l2res"] = timeit(us, torch.randint(0, 65536, (m,), device="cuda", dtype=torch.int32, generator=gen))
res["C_same"] = timeit(us, us.clone())
perm = torch.randperm(m, device="cuda", generator=gen)
res["D_shuffled"] = timeit(us[perm].contiguous(), vs[perm].contiguous())
for name, nbytes in (("copy32MiB", 32 << 20), ("copy1GiB", 1 << 30)):
    x = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        y.copy_(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(20):
        y.copy_(x)
    b.record(st)
    torch.cuda.synchronize()
    res[name + "_GBs"] = 2 * nbytes * 20 / (a.elapsed_time(b) / 1e3) / 1e9
res["m"] = m
for k in ("A_real", "B_l2res", "C_same", "D_shuffled"):
    res[k + "_GBs_rows"] = m * bits / 8 / (res[k] / 1e3) / 1e9
print(json.dumps(res), flush=True)
