"""CUDA-event timings of the raw builder C calls (outputs preallocated)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg
from paper_2208_11469_b200 import _native as N
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cache = f"/tmp/pg_rmat_{scale}_16_1.npz"
if os.path.exists(cache):
    z = np.load(cache); g = pg.CsrGraph(z["o"], z["a"])
else:
    g = pg.generate_kronecker(scale, 16, 1); np.savez(cache, o=g.offsets, a=g.adjacency)
d = g.device()
n = g.n
fam = pg.HashFamily(pg.DEFAULT_HASH_SEED, 32)
seeds = torch.from_numpy(fam.seeds_array().view(np.int64)).cuda()
st = torch.cuda.current_stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))
rows = torch.empty((n, 16), dtype=torch.int64, device="cuda"); ones = torch.empty(n, dtype=torch.int32, device="cuda")
ent = torch.empty((n, 64), dtype=torch.int32, device="cuda"); ln = torch.empty(n, dtype=torch.int32, device="cuda")
val = torch.empty((n, 64), dtype=torch.float64, device="cuda")
S = N.stream_handle()
res = {"scale": scale, "n": n, "nnz": d.nnz}
res["bloom1024"] = t(lambda: N.call("pg_build_bloom", N.ptr(d.offsets), N.ptr(d.adj), n, 1024, 2, N.ptr(seeds), N.ptr(rows), N.ptr(ones), S))
res["khash32"] = t(lambda: N.call("pg_build_khash", N.ptr(d.offsets), N.ptr(d.adj), n, 32, N.ptr(seeds), N.ptr(ent), S))
res["onehash64"] = t(lambda: N.call("pg_build_onehash", N.ptr(d.offsets), N.ptr(d.adj), n, 64, N.ptr(seeds), N.ptr(ent), N.ptr(ln), S))
res["kmv64"] = t(lambda: N.call("pg_build_kmv", N.ptr(d.offsets), N.ptr(d.adj), n, 64, N.ptr(seeds), N.ptr(val), N.ptr(ln), S))
res["python_build_bloom1024"] = t(lambda: pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=1024))
print(res, flush=True)
