#!/usr/bin/env python
"""Benchmark: edge-intersections/s of the fused Bloom triangle-count pass.

Workload (BASELINE.json configs[4], the metric's "1/2/4/8 B200" config; it
fits one GPU): R-MAT scale 24, edge factor 16, seed 4 (260.4 M undirected
edges), Bloom sketches B=2048, b=2, seed DEFAULT_HASH_SEED; one step = one
``tc_estimate(graph, sketched, "bf_and")`` pass over every edge of this
rank's shard (the fused gather + AND + popcount + histogram kernel) plus, for
N>1, the NCCL all-reduce of the popcount histogram.  The other configs are
parity-test cases (and ``secondary`` lines).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--gpus N`` outside torchrun re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU, 127.0.0.1 rendezvous).
One JSON line on rank 0.  ``--impl reference`` times the reference's CPU
algorithm on the host's cores: the graph from the oracle's C restatement of
the reference generator, Bloom rows from the oracle's C builder, and the
oracle's numpy port of the reference's chunked thread-pool pass -- no code of
the product package is imported on that arm.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOAD = {
    "c2": dict(desc="R-MAT s20 ef16 seed1 (a,b,c,d=.57,.19,.19,.05), Bloom B=1024 b=2, "
                    "tc_estimate bf_and", scale=20, ef=16, seed=1, bits=1024, b=2),
    "c5": dict(desc="R-MAT s24 ef16 seed4 (a,b,c,d=.57,.19,.19,.05), Bloom B=2048 b=2, "
                    "tc_estimate bf_and", scale=24, ef=16, seed=4, bits=2048, b=2),
}
METRIC = "edge-intersections/s (BF/MinHash TC) at 1/2/4/8 B200; % of HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(WORKLOAD), default="c5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-busy", action="store_true",
                    help="skip the untimed clock-sampling tail (for ncu runs)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the per-config measurements of configs 1-4 and 5b")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """Re-run this command under torch.distributed.run with n ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
           "--nproc-per-node", str(n), "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def config_dict(args, cfg, n, m):
    """The workload description both arms print (same keys and values)."""
    return {"workload": f"{args.config}: {cfg['desc']}", "n": int(n), "m": int(m),
            "sketch_bytes": int(n) * cfg["bits"] // 8,
            "l2": "flushed between timed steps (256 MiB write, outside the events); "
                  "the sketch matrix exceeds L2 at c5",
            "parallelism": (f"edge-range shards x{args.gpus}, replicated sketches, NCCL "
                            "all_reduce(int64[B+2])") if args.gpus > 1 else "1 GPU"}


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_profile(config: str) -> dict:
    """The committed ncu summary of this config's TC kernel (profiles/)."""
    path = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(config, {})
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# our arm


def run_ours(args, cfg, rank, world, local):
    import torch
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        # PG_BENCH_BACKEND=gloo: a functional check of the sharded path with
        # several ranks on one GPU (host-side all-reduce; not a measurement)
        backend = os.environ.get("PG_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, **({"device_id": torch.device("cuda", local)}
                                            if backend == "nccl" else {}))
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import _native as N
    from paper_2208_11469_b200.sharding import allreduce_counts, edge_range

    t0 = time.time()
    g = pg.generate_kronecker(cfg["scale"], cfg["ef"], cfg["seed"])  # on the device
    gen_s = time.time() - t0
    bits, b = cfg["bits"], cfg["b"]
    stream = torch.cuda.current_stream()

    # sketch build on the device (reported separately, not in the timed step)
    dev = g.device()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    build_ms = []
    for _ in range(3):
        ev0.record(stream)
        sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=b, bits_override=bits)
        ev1.record(stream)
        torch.cuda.synchronize()
        build_ms.append(ev0.elapsed_time(ev1))
    provider = pg.make_provider("bf_and", sketched=sk)
    m = g.m
    # the fused kernel's edge-slot layout
    t_lay = time.time()
    lay = provider._tc_layout(dev)
    torch.cuda.synchronize()
    layout_s = time.time() - t_lay
    lus, lvs, slots, padded = lay[:4]
    e_begin, e_end = edge_range(slots, rank, world, align=32 if padded else 1)
    rank_edges = int(((lvs[e_begin:e_end] != -1).sum()).item())
    layout_name = provider._tc_layout_name(lay)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def l2_flush():
        N.call("pg_l2_flush", N.ptr(flush), flush.numel(), N.stream_handle())

    def kernel():
        return provider._tc_counts_layout(lay, e_begin, e_end)

    def step():
        return allreduce_counts(kernel())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()

    # one CUDA graph per step (kernel + all-reduce: one launch, no host gaps)
    # and a kernel-only graph for the roofline's kernel time; eager if
    # capture fails (gloo)
    gstep = gkern = None
    graph_note = None
    try:
        gk, gs = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gk):
            kernel()
        with torch.cuda.graph(gs):
            step()
        gk.replay()
        gs.replay()
        torch.cuda.synchronize()
        gkern, gstep = gk, gs
    except Exception as exc:  # pragma: no cover - capture unsupported
        graph_note = f"eager ({type(exc).__name__}: capture failed)"
        torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kstarts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        time.sleep(0.2)
        if gstep is not None:
            # kernel-only replays first (roofline), then the K timed steps
            for i in range(args.steps):
                l2_flush()
                kstarts[i].record(stream)
                gkern.replay()
                kends[i].record(stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            for i in range(args.steps):
                l2_flush()  # between timed steps, outside the events
                starts[i].record(stream)
                gstep.replay()
                ends[i].record(stream)
        else:
            for i in range(args.steps):
                l2_flush()  # between timed steps, outside the events
                starts[i].record(stream)
                counts = kernel()
                kends[i].record(stream)
                counts = allreduce_counts(counts)
                ends[i].record(stream)
            kstarts = starts
        torch.cuda.synchronize()
        # keep the GPU busy for the clock sampler's benefit, untimed
        tq = time.time()
        while not args.no_busy and time.time() - tq < 0.5:
            kernel()
        torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kern_ms = [s.elapsed_time(e) for s, e in zip(kstarts, kends)]
    total_ms = sum(step_ms)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms, sum(kern_ms)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, kern_total = t.tolist()
    else:
        kern_total = sum(kern_ms)
    ms_per_step = total_ms / args.steps
    kern_ms_avg = kern_total / args.steps
    value = m / (ms_per_step / 1e3)  # whole-job edges per second

    counts = step().cpu().numpy()
    estimate = provider._tc_combine(counts) / 3.0

    # roofline of the dominant kernel.  achieved = the physical DRAM traffic
    # of one launch (committed ncu --set full capture of this config) over
    # the live kernel time; the algorithmic figure (two rows +
    # two int32 endpoints per edge, no reuse credit) is reported beside it.
    peak, peak_src = load_peaks()
    prof = load_profile(args.config) if world == 1 else {}
    bytes_per_edge = 2 * (bits // 8) + 8
    alg_gbs = rank_edges * bytes_per_edge / (kern_ms_avg / 1e3) / 1e9
    traffic = prof.get("dram_bytes_per_launch")
    phys_gbs = traffic / (kern_ms_avg / 1e3) / 1e9 if traffic else None
    roofline = {
        # the binding resource as the capture reports it (largest of DRAM
        # throughput, L2 throughput and the busiest SM pipe)
        "bound": prof.get("bound", "hbm"),
        "bound_pct": prof.get("bound_pct"),
        "top_pipes_pct": prof.get("top_pipes_pct"),
        "l2_throughput_pct": prof.get("l2_throughput_pct"),
        "dram_throughput_pct": prof.get("dram_throughput_pct"),
        "achieved": phys_gbs if phys_gbs is not None else alg_gbs,
        "peak": peak, "unit": "GB/s",
        "frac": (phys_gbs if phys_gbs is not None else alg_gbs) / peak,
        "traffic": traffic,
        "achieved_basis": ("physical: ncu dram bytes per launch / live kernel time"
                           if phys_gbs is not None else "algorithmic (no capture for this N)"),
        "kernel_ms": kern_ms_avg,
        "algorithmic": {"bytes_per_edge": bytes_per_edge, "edges_per_launch": rank_edges,
                        "effective_gbs": alg_gbs, "frac_of_peak": alg_gbs / peak},
        "l2_to_sm_bytes": prof.get("l2_to_sm_bytes"),
        "l2_to_sm_tbs": (prof["l2_to_sm_bytes"] / (kern_ms_avg / 1e3) / 1e12
                         if prof.get("l2_to_sm_bytes") else None),
        "capture": prof.get("source"),
        "peak_source": peak_src,
    }

    # e2e through the public API: pinned host CSR -> device sketches -> fused
    # pass -> host estimate, every step
    e2e = None
    if rank == 0 and world == 1 and args.e2e_steps > 0:
        e2e = run_e2e(pg, g, args.e2e_steps, bits, b, m)

    secondary = None
    if rank == 0 and world == 1 and not args.no_secondary:
        del sk, provider, lay, lus, lvs
        secondary = run_secondary(skip=args.config)

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(g, cfg, estimate)
        out = {
            "metric": METRIC, "value": value, "unit": "edge-intersections/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded R-MAT, the reference generator's draw order)",
            "config": config_dict(args, cfg, g.n, m),
            "layout": {"edges_per_rank": rank_edges, "edge_slots": slots,
                       "slot_range": [e_begin, e_end], "kind": layout_name,
                       "layout_build_s": layout_s},
            "roofline": roofline,
            "clocks": clk.summary(),
            # per timed step: the fused TC kernel (one graph replay) and the
            # L2-flush kernel between steps (outside the events, inside the
            # synchronised region)
            "gpu_launches": 2 * args.steps,
            "gpu_launches_per_step": {"tc_bloom_wide_kernel": 1, "l2_flush_kernel": 1},
            "cuda_graph": graph_note or "one graph replay per step (kernel + all-reduce)",
            "e2e": e2e,
            "cpu_baseline": cpu,
            "secondary": secondary,
            "estimate": estimate,
            "build": {"bloom_build_ms": min(build_ms), "graph_gen_s": gen_s,
                      "rows_per_s": g.n / (min(build_ms) / 1e3)},
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return out


def _time_device(fn, reps=5, warm=2, flush=None, graph=False):
    """Median CUDA-event time (ms) of fn() with an optional L2 flush before
    each timed call (outside the events); graph=True replays a CUDA graph of
    fn (launch-bound small configs)."""
    import torch
    st = torch.cuda.current_stream()
    out = None
    for _ in range(warm):
        out = fn()
    cg = None
    if graph:
        torch.cuda.synchronize()
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg):
            out = fn()
        cg.replay()
        torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        if cg is not None:
            cg.replay()
        else:
            out = fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out


def run_secondary(skip: str = "c5"):
    """The other BASELINE configs, one GPU: per-edge estimator throughput
    (device-resident inputs, L2 flushed before every timed call), each with
    the oracle port timed on a seeded sample of the same edges."""
    import gc
    import torch
    import paper_2208_11469_b200 as pg
    from paper_2208_11469_b200 import _native as N
    from paper_2208_11469_b200.mining import four_clique_counts, jaccard_counts, tc_counts
    peak, _ = load_peaks()
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def flush():
        N.call("pg_l2_flush", N.ptr(flush_buf), flush_buf.numel(), N.stream_handle())

    def rec(name, g, ms, bytes_per_edge, extra):
        r = {"graph": name, "n": g.n, "m": g.m, "ms": ms,
             "edge_intersections_per_s": g.m / (ms / 1e3),
             "algorithmic_gbs": g.m * bytes_per_edge / (ms / 1e3) / 1e9,
             "algorithmic_frac_of_hbm_peak": g.m * bytes_per_edge / (ms / 1e3) / 1e9 / peak}
        r.update(extra)
        return r

    from oracle import oracle as O
    port = O.NumpyPort(threads=len(os.sched_getaffinity(0)))

    def cpu_leg(g, p, chunk, sample):
        e = g.edges()
        rng = np.random.default_rng(0)
        idx = np.sort(rng.choice(len(e), size=min(sample, len(e)), replace=False))
        us, vs = e[idx, 0], e[idx, 1]
        t0 = time.perf_counter()
        cpu = port.tc_sum(chunk, us, vs)
        dt = time.perf_counter() - t0
        gpu = float(np.sum(p.pair_many(us, vs)))
        return {"cpu_edges_per_s": len(us) / dt, "cpu_sample_edges": int(len(us)),
                "cpu_cores": port.threads, "cpu_kind": "port", "speedup_vs_cpu": None,
                "cpu_gpu_sample_rel_err": abs(cpu - gpu) / max(1.0, abs(cpu))}

    def with_speedup(r, leg):
        leg["speedup_vs_cpu"] = r["edge_intersections_per_s"] / leg["cpu_edges_per_s"]
        r.update(leg)
        return r

    def bloom_tc(key, g, bits, b, sample):
        sk = pg.build_sketched_graph(g, "bloom", s=1.0, b=b, bits_override=bits)
        p = pg.make_provider("bf_and", sketched=sk)
        dev = g.device()
        p._tc_layout(dev)
        small = g.m < (1 << 20)
        ms, c = _time_device(lambda: tc_counts(p, dev), flush=flush, graph=small,
                             reps=20 if small else 5)
        r = rec(key, g, ms, 2 * bits // 8 + 8, {"estimate": p._tc_combine(c.cpu().numpy()) / 3.0})
        rows, sz = sk.bit_matrix, sk.sizes
        return with_speedup(r, cpu_leg(
            g, p, lambda a, b_: O.NumpyPort.bloom_chunk(rows, bits, b, "bf_and", sz, a, b_), sample))

    out = {}
    try:
        g = pg.generate_erdos_renyi_gnm(16384, 262144, 0)
        out["c1_bloom512_tc"] = bloom_tc("ER n=16384 m=262144 seed 0", g, 512, 1, 1 << 22)
        if skip != "c2":
            g = pg.generate_kronecker(20, 16, 1)
            out["c2_bloom1024_tc"] = bloom_tc("R-MAT s20 ef16 seed 1", g, 1024, 2, 1 << 22)
        # config 3: R-MAT s22 seed 2, 1-Hash k=64 and KMV k=64
        g = pg.generate_kronecker(22, 16, 2)
        for kind, bpe in (("onehash", 2 * 4 * 64 + 16), ("kmv", 2 * 8 * 64 + 24)):
            bms, sk = _time_device(lambda: pg.build_sketched_graph(g, kind, s=1.0, k_override=64),
                                   reps=1, flush=flush)
            p = pg.make_provider(kind, sketched=sk)
            torch.cuda.synchronize()
            t_lay = time.perf_counter()
            p._tc_layout(g.device())  # one-off edge-slot layout (cached on the graph / sketches)
            torch.cuda.synchronize()
            t_lay = time.perf_counter() - t_lay
            ms, c = _time_device(lambda: tc_counts(p, g.device()), reps=3, flush=flush)
            extra = {"estimate": p._tc_combine(c.cpu().numpy()) / 3.0, "build_ms": bms,
                     "layout_build_ms": t_lay * 1e3,
                     "layout": p._tc_layout_name(p._tc_layout(g.device()))}
            if kind == "kmv":
                kb = 2 * 4 * 64 + 24  # the rank kernels read 4-byte ranks
                extra.update(kernel_bytes_per_edge=kb,
                             frac_at_kernel_bytes=g.m * kb / (ms / 1e3) / 1e9 / peak,
                             engine="merge" if p._merge_engine() else "rank-directory")
            else:
                extra["rows"] = "hash-rank" if p._rank_rows() is not None else "id"
            r = rec("R-MAT s22 ef16 seed 2", g, ms, bpe, extra)
            sz = sk.sizes
            if kind == "onehash":
                ent = sk.entries
                chunk = lambda a, b_: O.NumpyPort.onehash_chunk(ent, 64, sz, a, b_)  # noqa: E731
                sample = 1 << 20
            else:
                vals, lens = sk.values, sk.lengths
                chunk = lambda a, b_: O.NumpyPort.kmv_chunk(vals, lens, 64, sz, a, b_)  # noqa: E731
                sample = 1 << 21
            out[f"c3_{kind}64_tc"] = with_speedup(r, cpu_leg(g, p, chunk, sample))
            del sk, p, chunk
        # config 4: Chung-Lu 2^23, k-Hash k=32 Jaccard >= 0.1
        g = pg.generate_chung_lu(1 << 23, 32, 2.1, 3)
        sk = pg.build_sketched_graph(g, "khash", s=1.0, k_override=32)
        ms, c = _time_device(lambda: jaccard_counts(g, sk, 0.1), flush=flush)
        c = c.cpu().numpy()
        r = rec("Chung-Lu n=2^23 avg 32 gamma 2.1 seed 3", g, ms, 2 * 4 * 32 + 8,
                {"kept_jhat_ge_0.1": int(c[0]), "kept_vertex_similarity_ge_0.1": int(c[1])})
        ent, sz = sk.entries, sk.sizes
        out["c4_khash32_jaccard"] = with_speedup(r, cpu_leg(
            g, pg.make_provider("khash", sketched=sk),
            lambda a, b_: O.NumpyPort.khash_chunk(ent, 32, sz, a, b_), 1 << 23))
        del sk, ent, g
        if skip != "c5":
            g = pg.generate_kronecker(24, 16, 4)
            out["c5_bloom2048_tc"] = bloom_tc("R-MAT s24 ef16 seed 4", g, 2048, 2, 1 << 23)
            del g
        gc.collect()
        torch.cuda.empty_cache()
        # config 5b: 4-clique, R-MAT s18 seed 4, Bloom 2048/2 over N+
        g = pg.generate_kronecker(18, 16, 4)
        view = pg.degree_order(g)
        dsk = pg.build_sketched_graph(g, "bloom", s=1.0, b=2, bits_override=2048,
                                      source="directed", view=view)
        p = pg.make_provider("bf_and", sketched=dsk)
        nnz = view.device().nnz
        ms, c = _time_device(lambda: four_clique_counts(view, p, 0, nnz), reps=3)
        c = c.cpu().numpy()
        r = {"graph": "R-MAT s18 ef16 seed 4", "ms": ms, "triples": int(c[-1]),
             "triples_per_s": int(c[-1]) / (ms / 1e3), "estimate": p._tc_combine(c[:-1])}
        # CPU: the C restatement (OpenMP, all host cores) over the fixed 1%
        # directed-edge sample (seed 0) of SURVEY 8(d)
        src = np.repeat(np.arange(view.n), view.out_degrees())
        ids = np.sort(np.random.default_rng(0).choice(len(src), size=len(src) // 100,
                                                      replace=False))
        O.C.set_threads(len(os.sched_getaffinity(0)))
        t0 = time.perf_counter()
        _, trip = O.C.four_clique_bloom(view.offsets, view.adjacency, dsk.bit_matrix, 2048, 2,
                                        edge_ids=ids)
        dt = time.perf_counter() - t0
        r.update({"cpu_triples_per_s": trip / dt, "cpu_sample_directed_edges": int(len(ids)),
                  "cpu_cores": len(os.sched_getaffinity(0)), "cpu_kind": "port (C oracle)",
                  "speedup_vs_cpu": r["triples_per_s"] / (trip / dt)})
        out["c5b_4clique_bloom2048"] = r
        # 4-clique with MinHash / KMV providers (k = 64, sketches over N+)
        from paper_2208_11469_b200.mining import four_clique_sketch_sum
        for kind in ("khash", "onehash", "kmv"):
            dsk = pg.build_sketched_graph(g, kind, s=1.0, k_override=64, source="directed",
                                          view=view)
            p = pg.make_provider(kind, sketched=dsk)
            ms, res = _time_device(lambda: four_clique_sketch_sum(view, p), reps=3)
            out[f"c5b_4clique_{kind}64"] = {"graph": "R-MAT s18 ef16 seed 4", "ms": ms,
                                             "triples": res[1], "estimate": res[0],
                                             "triples_per_s": res[1] / (ms / 1e3)}
            del dsk, p
    except Exception as exc:  # report, keep the headline line valid
        out["error"] = f"{type(exc).__name__}: {exc}"
    return out


def run_e2e(pg, g, steps, bits, b, m):
    """Same metric through the public API with HOST inputs every step.

    Input: the graph as a host int32 CSR in pinned memory (BASELINE's graph
    format).  Each step: CsrGraph(host arrays) -> build_sketched_graph (H2D of
    the CSR + device sketch build) -> tc_estimate (device edge slots, fused
    kernel, histogram D2H) -> float.
    """
    import torch

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    off_h = pinned(g.offsets)
    adj_h = pinned(g.adjacency.astype(np.int32))
    h2d = off_h.nbytes + adj_h.nbytes
    times, est = [], None
    for i in range(steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        graph = pg.CsrGraph(off_h, adj_h)
        skd = pg.build_sketched_graph(graph, "bloom", s=1.0, b=b, bits_override=bits)
        est = pg.tc_estimate(graph, skd, "bf_and")  # ends with the histogram D2H
        torch.cuda.synchronize()
        if i:  # first call is warm-up
            times.append(time.perf_counter() - t0)
        del graph, skd
    t = statistics.median(times)
    return {"value": m / t, "unit": "edge-intersections/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": 8 * (bits + 2), "ms_per_step": t * 1e3,
            "h2d_floor_ms": None,
            "path": "CsrGraph(pinned int32 CSR) -> build_sketched_graph(bloom, device) -> "
                    "tc_estimate(bf_and): chunked H2D of the CSR, per-chunk device sketch "
                    "build, device edge slots and fused kernel, histogram D2H, host combine",
            "estimate": est}


# ---------------------------------------------------------------------------
# CPU: the reference's algorithm on the host cores (oracle/ only)


def _cpu_rows(offsets, adjacency, bits, b):
    from oracle import oracle as O
    O.C.set_threads(len(os.sched_getaffinity(0)))
    rows, _ = O.C.build_bloom(offsets, adjacency, bits, b)
    return rows


def cpu_baseline(g, cfg, gpu_estimate, budget_s=12.0):
    """The oracle port of the reference's tc_estimate on all host cores over
    the same graph (rows from the C oracle builder, bit-identical to the
    device's): full passes until budget_s."""
    from oracle import oracle as O
    threads = len(os.sched_getaffinity(0))
    port = O.NumpyPort(threads=threads)
    bits, b = cfg["bits"], cfg["b"]
    rows = _cpu_rows(g.offsets, g.adjacency, bits, b)
    us, vs = O.upper_edges(g.offsets, g.adjacency)
    sizes = np.diff(g.offsets)

    def chunk(a, c):
        return O.NumpyPort.bloom_chunk(rows, bits, b, "bf_and", sizes, a, c)

    port.tc_sum(chunk, us[:1 << 18], vs[:1 << 18])  # warm-up
    passes, edges, t0 = 0, 0, time.perf_counter()
    full = None
    while True:
        full = port.tc_sum(chunk, us, vs) / 3.0
        passes += 1
        edges += len(us)
        if time.perf_counter() - t0 > budget_s or passes >= 3:
            break
    dt = time.perf_counter() - t0
    return {"value": edges / dt, "unit": "edge-intersections/s", "cores": threads,
            "kind": "port",
            "sample": f"{passes} full tc_estimate pass(es) over all {len(us)} edges "
                      "(numpy port of the reference's chunked thread-pool path)",
            "estimate": full,
            "parity_rel_err_vs_gpu": abs(full - gpu_estimate) / max(1.0, abs(full))}


def run_reference(args, cfg, rank, world):
    """The reference's CPU path on this host, without the product package:
    graph = oracle C restatement of generate_kronecker (bit-identical, pinned
    in tests), rows = oracle C Bloom builder, each step = the numpy port of
    BloomProvider.pair_many + _chunked_sum over a seeded 2^24-edge slice."""
    if rank != 0:
        return None
    from oracle import oracle as O
    threads = len(os.sched_getaffinity(0))
    O.C.set_threads(threads)
    port = O.NumpyPort(threads=threads)
    t0 = time.time()
    off, adj = O.C.generate_kronecker(cfg["scale"], cfg["ef"], cfg["seed"])
    gen_s = time.time() - t0
    bits, b = cfg["bits"], cfg["b"]
    t0 = time.time()
    rows, _ = O.C.build_bloom(off, adj, bits, b)
    build_s = time.time() - t0
    us, vs = O.upper_edges(off, adj)
    sizes = np.diff(off)
    n, m = len(off) - 1, len(us)
    sample = min(m, 1 << 24)

    def chunk(a, c):
        return O.NumpyPort.bloom_chunk(rows, bits, b, "bf_and", sizes, a, c)

    rng = np.random.default_rng(0)
    starts = rng.integers(0, max(1, m - sample), size=args.warmup + args.steps)
    for i in range(args.warmup):
        s0 = int(starts[i])
        port.tc_sum(chunk, us[s0:s0 + sample], vs[s0:s0 + sample])
    times = []
    for i in range(args.steps):
        s0 = int(starts[args.warmup + i])
        t1 = time.perf_counter()
        port.tc_sum(chunk, us[s0:s0 + sample], vs[s0:s0 + sample])
        times.append(time.perf_counter() - t1)
    ms = 1e3 * sum(times) / len(times)
    value = sample / (ms / 1e3)
    out = {"metric": METRIC, "value": value, "unit": "edge-intersections/s", "impl": "reference",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
           "data": "synthetic (seeded R-MAT, the reference generator's draw order)",
           "config": config_dict(args, cfg, n, m),
           "cpu_baseline": {"value": value, "unit": "edge-intersections/s", "cores": threads,
                            "kind": "port",
                            "sample": f"per step a contiguous {sample}-edge slice of the "
                                      "upper edge list at a seeded random offset (seed 0); "
                                      "numpy port of BloomProvider.pair_many + _chunked_sum"},
           "e2e": {"value": value, "unit": "edge-intersections/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "setup": {"graph_gen_s": gen_s, "bloom_build_s": build_s,
                     "graph": "oracle C generate_kronecker (pgo_rmat_pairs + "
                              "pgo_csr_from_pairs), rows from pgo_build_bloom"}}
    print(json.dumps(out), flush=True)
    return out


def main():
    args = parse()
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    cfg = WORKLOAD[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    run_ours(args, cfg, rank, world, local)


if __name__ == "__main__":
    main()
