set -x
timeout 900 python -m pytest tests/test_gpu_kmv_ranked.py tests/test_gpu_determinism.py tests/test_gpu_large.py -q -x > gpurun_out/t_af.log 2>&1; echo rc=$? >> gpurun_out/t_af.log
for e in h d h; do PG_KMV_ENGINE=$e timeout 300 python scripts/time_kernels.py c3kmv >> gpurun_out/time_af.log 2>&1; done
tail -15 gpurun_out/t_af.log; cat gpurun_out/time_af.log
