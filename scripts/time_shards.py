"""Per-shard kernel time of the fused passes when the edge slots are split
into N shares (provider._tc_counts_shard, as tc_counts(rank, world) does):
the load balance of a multi-GPU run, measured on one GPU."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg  # noqa: E402

W = int(os.environ.get("PG_SHARDS", "8"))


def shard_times(p, dev, label):
    lay = p._tc_layout(dev)
    ts = []
    for r in range(W):
        p._tc_counts_shard(lay, r, W)
        torch.cuda.synchronize()
        vals = []
        for _ in range(3):
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            p._tc_counts_shard(lay, r, W)
            z.record()
            torch.cuda.synchronize()
            vals.append(a.elapsed_time(z))
        ts.append(statistics.median(vals))
    print(f"{label}: shards(ms) {[round(t, 3) for t in ts]}  max/mean {max(ts) / (sum(ts) / W):.3f}",
          flush=True)


for cfg in sys.argv[1:]:
    if cfg == "c5":
        g = pg.generate_kronecker(24, 16, 4)
        sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048)
        shard_times(pg.make_provider("bf_and", sketched=sk), g.device(), "c5 bloom")
    elif cfg == "c3":
        g = pg.generate_kronecker(22, 16, 2)
        for kind in ("onehash", "kmv"):
            sk = pg.build_sketched_graph(g, kind, s=1.0, k_override=64)
            shard_times(pg.make_provider(kind, sketched=sk), g.device(), f"c3 {kind}")
            del sk
