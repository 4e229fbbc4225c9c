"""Golden values of the reference's sampling TC baselines (build container only).

    python tests/golden/make_golden_baselines.py

doulion_tc and reduced_execution_tc (reference mining.py:334-367) on seeded
graphs for several probabilities / fractions and seeds.  Writes
baselines.json.  Nothing at test time reads /root/reference.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import probgraph as R  # noqa: E402
from paper_2208_11469_b200 import graphs as G  # noqa: E402

out = {}
for name, mine in (("rmat12", G.generate_kronecker(12, 16, 8, device=False)),
                   ("er2000", G.generate_erdos_renyi_gnm(2000, 30000, 9))):
    g = R.CsrGraph(mine.offsets, mine.adjacency.astype(np.int64))
    view = R.degree_order(g)
    rec = {"n": g.n, "m": g.m, "doulion": {}, "reduced": {}}
    for p in (1.0, 0.5, 0.25):
        for seed in (0, 7):
            rec["doulion"][f"{p}/{seed}"] = R.doulion_tc(g, p, seed)
    for f in (1.0, 0.3, 0.05):
        for seed in (0, 7):
            rec["reduced"][f"{f}/{seed}"] = R.reduced_execution_tc(view, f, seed)
    out[name] = rec
    print(name, rec["doulion"]["1.0/0"], flush=True)
json.dump(out, open(os.path.join(HERE, "baselines.json"), "w"), indent=1)
