set -x
timeout 900 python -m pytest tests/test_gpu_generators.py tests/test_gpu_clique_sketch.py tests/test_gpu_large.py -q -x > gpurun_out/t_ap.log 2>&1; echo rc=$? >> gpurun_out/t_ap.log
timeout 600 python -c "
import time, torch, sys
sys.path.insert(0, '.')
import paper_2208_11469_b200 as pg
g = pg.generate_kronecker(24, 16, 4)
dev = g.device(); torch.cuda.synchronize()
for i in range(3):
    dev._layouts.clear()
    t = time.perf_counter(); r = dev.degree_rank(); torch.cuda.synchronize(); print('degree_rank s24', (time.perf_counter()-t)*1e3, 'ms')
" > gpurun_out/dr_ap.log 2>&1
tail -3 gpurun_out/t_ap.log; cat gpurun_out/dr_ap.log
