"""The edge-range sharder with the real device kernels: two ranks, both on
cuda:0 (a functional check -- the all-reduce is gloo's host-side one, so no
rank waits on another's kernel), each runs the fused pass over its share of
the padded edge slots (mining.tc_counts(rank, world)) and
sharding.tc_estimate_sharded sums the integer partials.  Every estimator
kind must reproduce the single-process estimate (bit-identical integer
partials; KMV's fp64 sum to 1e-12)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

KINDS = [("bloom", "bf_and", {"b": 2, "bits_override": 1024}),
         ("bloom", "bf_or", {"b": 1, "bits_override": 512}),
         ("khash", "khash", {"k_override": 32}),
         ("onehash", "onehash", {"k_override": 64}),
         ("kmv", "kmv", {"k_override": 64})]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _clique_args(pg, g):
    view = pg.degree_order(g)
    dsk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048, source="directed", view=view)
    return view, pg.make_provider("bf_and", sketched=dsk)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200.sharding import four_clique_count_sharded, tc_estimate_sharded
    g = pg.generate_kronecker(14, 16, 9)
    out = {}
    for sk_kind, kind, kw in KINDS:
        sk = pg.build_sketched_graph(g, sk_kind, s=1.0, **kw)
        out[kind] = tc_estimate_sharded(g, sk, kind)
    out["4clique"] = four_clique_count_sharded(*_clique_args(pg, g))
    dist.destroy_process_group()
    q.put((rank, out))


def test_two_ranks_one_gpu_match_single_process():
    import paper_2208_11469_b200 as pg
    g = pg.generate_kronecker(14, 16, 9)
    want = {}
    for sk_kind, kind, kw in KINDS:
        want[kind] = pg.tc_estimate(g, pg.build_sketched_graph(g, sk_kind, s=1.0, **kw), kind)
    want["4clique"] = pg.four_clique_count(*_clique_args(pg, g))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        for kind, v in want.items():
            if kind == "kmv":
                assert res[r][kind] == pytest.approx(v, rel=1e-12), (r, kind)
            else:
                assert res[r][kind] == v, (r, kind)
