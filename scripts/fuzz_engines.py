"""Differential fuzz of the c3 engines: random graphs, k and seeds; the
hash-rank 1-Hash engine against the ID-row engine (identical integers) and
the KMV merge engine against the rank-directory and values engines
(|rel| <= 1e-12), whole graph and random shard splits.

    python scripts/fuzz_engines.py [seconds]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402
from paper_2208_11469_b200 import _native as N  # noqa: E402
from paper_2208_11469_b200.mining import tc_counts  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(12345)
t0 = time.time()
cases = 0


def graph(kind):
    if kind == 0:
        return pg.generate_kronecker(int(rng.integers(6, 15)), int(rng.integers(2, 24)), int(rng.integers(1, 1 << 20)))
    if kind == 1:
        n = int(rng.integers(10, 4000))
        m = int(rng.integers(1, min(n * (n - 1) // 2, 40 * n) + 1))
        return pg.generate_erdos_renyi_gnm(n, m, int(rng.integers(1, 1 << 20)))
    # hubs over a sparse background, isolated vertices at the end
    n = int(rng.integers(50, 3000))
    hubs = int(rng.integers(1, 6))
    e = [[h, int(x)] for h in range(hubs) for x in rng.choice(np.arange(hubs, n - 5), size=int(rng.integers(1, n - hubs - 5)), replace=False)]
    e += [[int(a), int(b)] for a, b in rng.integers(hubs, n - 5, size=(int(rng.integers(1, 4 * n)), 2)) if a != b]
    return pg.CsrGraph.from_edges(e, n)


def counts(p, dev, world):
    if world == 1:
        return tc_counts(p, dev).cpu().numpy()
    return sum(tc_counts(p, dev, r, world).cpu().numpy() for r in range(world))


while time.time() - t0 < budget:
    g = graph(int(rng.integers(0, 3)))
    if g.m == 0:
        continue
    k = int(rng.choice([32, 64, 128]))
    dev = g.device()
    world = int(rng.choice([1, 2, 3, 5]))
    for var in ("PG_KMV_ENGINE", "PG_ONEHASH_ROWS", "PG_TC_ORIENT", "PG_ONEHASH_LAYOUT", "PG_KMV_PARTITION"):
        os.environ.pop(var, None)
    # ---- 1-Hash
    sk = pg.build_sketched_graph(g, "onehash", s=1.0, k_override=k)
    if rng.random() < 0.3:
        os.environ["PG_TC_ORIENT"] = "id"
    if rng.random() < 0.2:
        os.environ["PG_ONEHASH_LAYOUT"] = "plain"
    p = pg.make_provider("onehash", sketched=sk)
    got = counts(p, dev, world)
    os.environ["PG_ONEHASH_ROWS"] = "id"
    want = counts(pg.make_provider("onehash", sketched=sk), dev, 1)
    assert np.array_equal(got, want), ("onehash", g.n, g.m, k, world, dict(os.environ))
    for var in ("PG_ONEHASH_ROWS", "PG_TC_ORIENT", "PG_ONEHASH_LAYOUT"):
        os.environ.pop(var, None)
    # ---- KMV
    sk = pg.build_sketched_graph(g, "kmv", s=1.0, k_override=k)
    if rng.random() < 0.3:
        os.environ["PG_TC_ORIENT"] = "id"
    if rng.random() < 0.2:
        os.environ["PG_KMV_PARTITION"] = "0"
    p = pg.make_provider("kmv", sketched=sk)
    got = float(counts(p, dev, world)[0])
    os.environ["PG_KMV_ENGINE"] = "ranked"
    sk._kmv_merge_layout = None
    ranked = float(counts(pg.make_provider("kmv", sketched=sk), dev, 1)[0])
    us, vs = dev.upper_edges()
    d = sk.device_tensors()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    N.call("pg_tc_kmv", N.ptr(d["values"]), N.ptr(d["lengths"]), k, N.ptr(d["sizes"]), N.ptr(us), N.ptr(vs),
           0, us.numel(), N.ptr(out), N.stream_handle())
    values = float(out.item())
    tol = 1e-12 * max(1.0, abs(values))
    assert abs(got - values) <= tol and abs(ranked - values) <= tol, ("kmv", g.n, g.m, k, world, got, ranked, values)
    cases += 1
print(f"fuzz ok: {cases} graphs in {time.time() - t0:.0f} s", flush=True)
