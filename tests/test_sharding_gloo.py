"""Multi-rank host logic of the edge-range sharder on CPU (gloo, world 2).

Each rank computes the integer partials of ITS edge range in exactly the
layout the device kernels emit ([hist(B+1), sum_pos] for Bloom,
[cnt(k+1), ssum(k+1), verbatim] for MinHash), the partials are summed with
``allreduce_counts`` over gloo, and the combined estimate must equal the
single-process result (bit-identical histograms, estimate to 1e-12).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup():
    import paper_2208_11469_b200 as pg
    g = pg.generate_kronecker(12, 8, 5)
    us, vs = O.upper_edges(g.offsets, g.adjacency)
    return pg, g, us, vs


def _bloom_partials(g, us, vs, lo, hi, bits, b, kind):
    rows, ones = O.C.build_bloom(g.offsets, g.adjacency, bits, b)
    sizes = np.diff(g.offsets)
    a, c = us[lo:hi], vs[lo:hi]
    pop = O.C.pairs_bloom(rows, bits, kind == "bf_or", a, c)
    if kind == "bf_or":
        S = sizes[a] + sizes[c]
        lut = O.swamidass(bits, b, np.arange(bits + 1))
        pos = (S - lut[pop]) > 0
        hist = np.bincount(pop[pos], minlength=bits + 1)
        return np.concatenate([hist, [int(S[pos].sum())]]).astype(np.int64), rows, ones
    return np.concatenate([np.bincount(pop, minlength=bits + 1), [0]]).astype(np.int64), rows, ones


def _minhash_partials(g, us, vs, lo, hi, k, onehash):
    sizes = np.diff(g.offsets)
    if onehash:
        ent, _ = O.C.build_onehash(g.offsets, g.adjacency, k)
    else:
        ent = O.C.build_khash(g.offsets, g.adjacency, k)
    a, c = us[lo:hi], vs[lo:hi]
    m = O.C.pairs_minhash(ent, k, onehash, a, c)
    S = sizes[a] + sizes[c]
    verb = (sizes[a] <= k) & (sizes[c] <= k) if onehash else np.zeros(len(a), bool)
    cnt = np.bincount(m[~verb], minlength=k + 1)
    ssum = np.bincount(m[~verb], weights=S[~verb], minlength=k + 1).astype(np.int64)
    return np.concatenate([cnt, ssum, [int(m[verb].sum())]]).astype(np.int64), ent


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2208_11469_b200.sharding import allreduce_counts, edge_range
    from paper_2208_11469_b200.providers import BloomProvider, MinHashProvider
    from paper_2208_11469_b200.sketches import BudgetPlan, SketchedGraph
    pg, g, us, vs = _setup()
    lo, hi = edge_range(len(us), rank, world)
    out = {}
    for kind in ("bf_and", "bf_l", "bf_or"):
        part, rows, ones = _bloom_partials(g, us, vs, lo, hi, 512, 2, kind)
        t = allreduce_counts(torch.from_numpy(part))
        sk = SketchedGraph("bloom", BudgetPlan.explicit("bloom", g.n, bits=512, b=2),
                           pg.HashFamily(pg.DEFAULT_HASH_SEED, 2), "undirected",
                           np.diff(g.offsets), bit_matrix=rows, ones=ones)
        out[kind] = (t.numpy().tolist(), BloomProvider(sk, kind)._tc_combine(t.numpy()) / 3.0)
    for kind, onehash in (("khash", False), ("onehash", True)):
        part, ent = _minhash_partials(g, us, vs, lo, hi, 16, onehash)
        t = allreduce_counts(torch.from_numpy(part))
        sk = SketchedGraph(kind, BudgetPlan.explicit(kind, g.n, k=16),
                           pg.HashFamily(pg.DEFAULT_HASH_SEED, 16 if not onehash else 1),
                           "undirected", np.diff(g.offsets), entries=ent,
                           lengths=np.minimum(np.diff(g.offsets), 16))
        out[kind] = (t.numpy().tolist(), MinHashProvider(sk)._tc_combine(t.numpy()) / 3.0)
    results[rank] = out
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_allreduce_matches_single_process():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    pg, g, us, vs = _setup()
    sizes = np.diff(g.offsets)
    full = {}
    for kind in ("bf_and", "bf_l", "bf_or"):
        part, rows, _ = _bloom_partials(g, us, vs, 0, len(us), 512, 2, kind)
        est = O.NumpyPort(threads=1).tc_sum(
            lambda a, c: O.NumpyPort.bloom_chunk(rows, 512, 2, kind, sizes, a, c), us, vs) / 3.0
        full[kind] = (part.tolist(), est)
    for kind, onehash in (("khash", False), ("onehash", True)):
        part, ent = _minhash_partials(g, us, vs, 0, len(us), 16, onehash)
        fn = O.NumpyPort.onehash_chunk if onehash else O.NumpyPort.khash_chunk
        est = O.NumpyPort(threads=1).tc_sum(lambda a, c: fn(ent, 16, sizes, a, c), us, vs) / 3.0
        full[kind] = (part.tolist(), est)
    for rank in range(world):
        for kind, (counts, est) in results[rank].items():
            assert counts == full[kind][0], kind
            assert est == pytest.approx(full[kind][1], rel=1e-12), kind
