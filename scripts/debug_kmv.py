import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2208_11469_b200 as pg
z = np.load("tests/golden/small_cases.npz")
name, k = sys.argv[1], int(sys.argv[2])
g = pg.CsrGraph(z[f"{name}/offsets"], z[f"{name}/adjacency"])
seed = {"g60": 4, "g80": 6, "g200": 42, "dense120": 7, "sparse300": 11}[name] + 300
sk = pg.build_sketched_graph(g, "kmv", s=1.0, seed=seed, k_override=k)
print("built", flush=True)
e = g.edges()
p = pg.make_provider("kmv", sketched=sk)
est = p.pair_many(e[:, 0], e[:, 1])
print("pairs", np.array_equal(est, z[f"{name}/kmv{k}/pairs"]), flush=True)
print("tc", pg.tc_estimate(g, sk, "kmv"), z[f"{name}/kmv{k}/tc"][0], flush=True)
jp = pg.jarvis_patrick_cluster(g, p, 1.0)
print("jp", [len(jp.kept_edges), jp.cluster_count, jp.singleton_count], z[f"{name}/kmv{k}/jp"].tolist(), flush=True)
