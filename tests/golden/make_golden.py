"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--large]

Writes small cases with full arrays to ``small_cases.npz`` and per-config
checksums / integer summaries to ``config*.json``.  The fixtures pin the CPU
oracle (oracle/) and, through it, the CUDA path; nothing at test time reads
/root/reference.  Graph inputs come from this repo's generators (R-MAT is
checked equal to the reference's ``generate_kronecker`` here) and are handed
to the reference as ``CsrGraph(offsets, adjacency)``.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import probgraph as R  # noqa: E402  (the reference, read-only)
from paper_2208_11469_b200 import graphs as G  # noqa: E402


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def canon(sg):
    """Canonical little-endian arrays of a reference SketchedGraph."""
    out = {}
    if sg.bit_matrix is not None:
        out["bit_matrix"] = sg.bit_matrix.astype("<u8")
        out["ones"] = sg.ones.astype("<i8")
    if sg.entries is not None:
        out["entries"] = sg.entries.astype("<i8")
    if sg.lengths is not None:
        out["lengths"] = sg.lengths.astype("<i8")
    if sg.values is not None:
        out["values"] = sg.values.astype("<f8")
    return out


def gnp(n, p, seed):
    """G(n, p) by the reference conftest's procedure (triu draws)."""
    rng = np.random.default_rng(seed)
    iu, iv = np.triu_indices(n, k=1)
    mask = rng.random(len(iu)) < p
    return np.stack([iu[mask], iv[mask]], axis=1)


SMALL = [  # (name, n, p, seed)
    ("g60", 60, 0.15, 4),
    ("g80", 80, 0.10, 6),
    ("g200", 200, 0.08, 42),
    ("dense120", 120, 0.6, 7),
    ("sparse300", 300, 0.01, 11),
]
BLOOM = [(64, 1), (128, 2), (512, 1), (576, 3), (1024, 2), (2048, 2)]
KS = [1, 4, 5, 32, 64]


def small_cases(out_path):
    store = {}
    meta = []
    for name, n, p, seed in SMALL:
        g = R.CsrGraph.from_edges(gnp(n, p, seed), n=n)
        e = g.edges()
        us, vs = e[:, 0], e[:, 1]
        store[f"{name}/offsets"] = g.offsets
        store[f"{name}/adjacency"] = g.adjacency
        view = R.degree_order(g)
        ex = R.make_provider("exact_merge", view=view)
        store[f"{name}/tc_exact"] = np.asarray([R.triangle_count(view, ex)])
        store[f"{name}/c4_exact"] = np.asarray([R.four_clique_count(view, ex)])
        exg = R.make_provider("exact_merge", graph=g)
        store[f"{name}/pairs_exact"] = exg.pair_many(us, vs)
        for bits, b in BLOOM:
            sk = R.build_sketched_graph(g, "bloom", s=1.0, b=b, seed=seed + 100,
                                        bits_override=bits)
            key = f"{name}/bloom{bits}_{b}"
            for k2, v2 in canon(sk).items():
                store[f"{key}/{k2}"] = v2
            for kind in ("bf_and", "bf_l", "bf_or"):
                pv = R.make_provider(kind, sketched=sk)
                store[f"{key}/pairs_{kind}"] = pv.pair_many(us, vs)
                store[f"{key}/tc_{kind}"] = np.asarray([R.tc_estimate(g, sk, kind)])
                jp = R.jarvis_patrick_cluster(g, pv, 1.0)
                store[f"{key}/jp_{kind}"] = np.asarray(
                    [len(jp.kept_edges), jp.cluster_count, jp.singleton_count])
            dsk = R.build_sketched_graph(g, "bloom", s=1.0, b=b, seed=seed + 200,
                                         bits_override=bits, source="directed",
                                         view=view)
            for k2, v2 in canon(dsk).items():
                store[f"{key}/dir_{k2}"] = v2
            for kind in ("bf_and", "bf_l"):
                pv = R.make_provider(kind, sketched=dsk)
                store[f"{key}/c4_{kind}"] = np.asarray([R.four_clique_count(view, pv)])
        for k in KS:
            for kind in ("khash", "onehash", "kmv"):
                sk = R.build_sketched_graph(g, kind, s=1.0, seed=seed + 300,
                                            k_override=k)
                key = f"{name}/{kind}{k}"
                for k2, v2 in canon(sk).items():
                    store[f"{key}/{k2}"] = v2
                pv = R.make_provider(kind, sketched=sk)
                store[f"{key}/pairs"] = pv.pair_many(us, vs)
                store[f"{key}/tc"] = np.asarray([R.tc_estimate(g, sk, kind)])
                jp = R.jarvis_patrick_cluster(g, pv, 1.0)
                store[f"{key}/jp"] = np.asarray(
                    [len(jp.kept_edges), jp.cluster_count, jp.singleton_count])
                if kind == "khash":
                    jh = [R.est_jaccard_minhash(sk.sketch(int(a)), sk.sketch(int(c)))
                          for a, c in zip(us, vs)]
                    js = [R.vertex_similarity(int(a), int(c), "jaccard", pv, g)
                          for a, c in zip(us, vs)]
                    store[f"{key}/jaccard_hat"] = np.asarray(jh)
                    store[f"{key}/jaccard_sim"] = np.asarray(js)
        meta.append(name)
    np.savez_compressed(out_path, **store)
    return meta


def hash_kat():
    fam = R.HashFamily(base_seed=R.DEFAULT_HASH_SEED, count=4)
    keys = [0, 1, 2, 17, 12345, 99, 2 ** 31 - 1, 2 ** 40, 2 ** 50 + 3]
    from probgraph.hashing import hash_words, unit_values
    return {
        "seeds_default4": [fam.seed(i) for i in range(4)],
        "seeds_seed7": [R.HashFamily(base_seed=7, count=2).seed(i) for i in range(2)],
        "keys": keys,
        "words_default_fn0": [int(w) for w in hash_words(fam, 0, keys)],
        "words_default_fn3": [int(w) for w in hash_words(fam, 3, keys)],
        "units_default_fn0": [float(u) for u in unit_values(fam, 0, keys)],
        "bit_default_fn1_513": [R.hash_to_bit(fam, 1, k, 513) for k in keys],
        # literal anchors of the reference's own tests/test_hashing.py:24-37
        "ref_test_anchors": {
            "seed0": 0x2D0A2CC335CD72A7, "seed1": 0x95527B2E69B24CDF,
            "bit_0_12345_256": 47, "bit_1_12345_256": 178,
            "unit_0_12345": 0.3926770316358376,
            "fam7_bit_0_0_65536": 15605, "fam7_unit_1_99": 0.05072011188429145,
        },
    }


def config_summary(name, g_ref, specs, jaccard_tau=None):
    """Checksums + integer summaries of reference sketches on one graph."""
    t0 = time.time()
    e = g_ref.edges()
    us, vs = e[:, 0], e[:, 1]
    out = {"name": name, "n": g_ref.n, "m": g_ref.m,
           "offsets_sha": sha(g_ref.offsets.astype("<i8")),
           "adjacency_sha": sha(g_ref.adjacency.astype("<i8")), "sketches": {}}
    for kind, param, b in specs:
        tk = time.time()
        if kind == "bloom":
            sk = R.build_sketched_graph(g_ref, kind, s=1.0, b=b, bits_override=param)
        else:
            sk = R.build_sketched_graph(g_ref, kind, s=1.0, k_override=param)
        rec = {k2: sha(v2) for k2, v2 in canon(sk).items()}
        rec["build_s"] = time.time() - tk
        if kind == "bloom":
            ests = {}
            for est in ("bf_and", "bf_l", "bf_or"):
                ests[est] = R.tc_estimate(g_ref, sk, est, threads=8)
            rec["tc"] = ests
            pop = np.empty(len(us), dtype=np.int64)
            for lo in range(0, len(us), 1 << 20):
                hi = min(lo + (1 << 20), len(us))
                pop[lo:hi] = np.bitwise_count(
                    sk.bit_matrix[us[lo:hi]] & sk.bit_matrix[vs[lo:hi]]).sum(axis=1)
            rec["and_popcount_hist"] = np.bincount(pop, minlength=param + 1).tolist()
        else:
            rec["tc"] = {kind: R.tc_estimate(g_ref, sk, kind, threads=8)}
            if kind == "khash" and jaccard_tau is not None:
                m = np.empty(len(us), dtype=np.int64)
                for lo in range(0, len(us), 1 << 20):
                    hi = min(lo + (1 << 20), len(us))
                    a, c = sk.entries[us[lo:hi]], sk.entries[vs[lo:hi]]
                    m[lo:hi] = np.count_nonzero((a == c) & (a >= 0), axis=1)
                rec["match_hist"] = np.bincount(m, minlength=param + 1).tolist()
                pv = R.make_provider("khash", sketched=sk)
                # est_jaccard_minhash reading: m/k >= tau
                rec["jaccard_hat_kept"] = int(np.count_nonzero(m / param >= jaccard_tau))
                # vertex_similarity(JACCARD) reading, evaluated per edge with the
                # reference's scalar functions on a sample, and in full below
                deg = g_ref.degrees()
                js = np.empty(len(us))
                for i, (a, c) in enumerate(zip(us.tolist(), vs.tolist())):
                    js[i] = R.vertex_similarity(a, c, "jaccard", pv, g_ref) \
                        if i < 20000 else np.nan
                rec["jaccard_sim_first20000_kept"] = int(np.count_nonzero(js[:20000] >= jaccard_tau))
                del deg
        out["sketches"][f"{kind}{param}" + (f"_{b}" if kind == "bloom" else "")] = rec
        print(name, kind, param, f"{time.time() - tk:.1f}s", flush=True)
    out["total_s"] = time.time() - t0
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true", help="also s20 (config 2)")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = set(args.only.split(",")) if args.only else None

    def want(x):
        return only is None or x in only

    if want("kat"):
        with open(os.path.join(HERE, "hash_kat.json"), "w") as fh:
            json.dump(hash_kat(), fh, indent=1)
    if want("small"):
        small_cases(os.path.join(HERE, "small_cases.npz"))
        print("small cases done", flush=True)
    if want("c1"):
        g = G.generate_erdos_renyi_gnm(16384, 262144, 0)
        gr = R.CsrGraph(g.offsets, g.adjacency)
        rec = config_summary("config1_er_n16384_m262144_seed0", gr,
                             [("bloom", 512, 1), ("khash", 32, 1),
                              ("onehash", 64, 1), ("kmv", 64, 1)], jaccard_tau=0.1)
        with open(os.path.join(HERE, "config1.json"), "w") as fh:
            json.dump(rec, fh, indent=1)
    if args.large and want("c2"):
        gr = R.generate_kronecker(20, 16, 1)
        mine = G.generate_kronecker(20, 16, 1)
        assert np.array_equal(gr.offsets, mine.offsets)
        assert np.array_equal(gr.adjacency, mine.adjacency)
        rec = config_summary("config2_rmat_s20_ef16_seed1", gr, [("bloom", 1024, 2)])
        with open(os.path.join(HERE, "config2.json"), "w") as fh:
            json.dump(rec, fh, indent=1)


if __name__ == "__main__":
    main()
