"""CUDA-event timing of the sketch builders at the BASELINE configs (dev tool)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


cases = [("c2", lambda: pg.generate_kronecker(20, 16, 1), [("bloom", dict(b=2, bits_override=1024))]),
         ("c3", lambda: pg.generate_kronecker(22, 16, 2), [("onehash", dict(k_override=64)), ("kmv", dict(k_override=64))]),
         ("c4", lambda: pg.generate_chung_lu(1 << 23, 32, 2.1, 3), [("khash", dict(k_override=32))]),
         ("c5", lambda: pg.generate_kronecker(24, 16, 4), [("bloom", dict(b=2, bits_override=2048))])]
for name, mk, kinds in cases:
    if len(sys.argv) > 1 and name not in sys.argv[1:]:
        continue
    g = mk()
    g.device()
    for kind, kw in kinds:
        t = timed(lambda: pg.build_sketched_graph(g, kind, s=1.0, **kw))
        print(f"{name} {kind} {kw}: {t:.2f} ms  n={g.n} entries={int(g.offsets[-1])}  "
              f"{int(g.offsets[-1]) / t / 1e6:.1f} G entries/s", flush=True)
    del g
