"""k-Hash TC and Jaccard-count timings (dev tool): s20 k=32/64, c4-shape."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2208_11469_b200 as pg
from paper_2208_11469_b200.mining import tc_counts, jaccard_counts

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): out = fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out

g = pg.generate_kronecker(20, 16, 1)
for k in (32, 64):
    sk = pg.build_sketched_graph(g, "khash", s=1.0, k_override=k)
    p = pg.make_provider("khash", sketched=sk)
    ms, c = t(lambda: tc_counts(p, g.device()))
    ms2, j = t(lambda: jaccard_counts(g, sk, 0.1))
    print(f"s20 k={k} tc {ms:.3f} ms jaccard {ms2:.3f} ms", p._tc_combine(c.cpu().numpy()), j[:2].tolist())
g = pg.generate_chung_lu(1 << 23, 32, 2.1, 3)
sk = pg.build_sketched_graph(g, "khash", s=1.0, k_override=32)
ms2, j = t(lambda: jaccard_counts(g, sk, 0.1))
print(f"c4 jaccard {ms2:.3f} ms", j[:2].tolist())
