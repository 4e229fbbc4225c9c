set -x
timeout 900 python -m pytest tests/test_gpu_guards.py tests/test_gpu_determinism.py tests/test_gpu_e2e.py tests/test_gpu_kmv_ranked.py -q > gpurun_out/t_k.log 2>&1; echo rc=$? >> gpurun_out/t_k.log
timeout 300 python scripts/time_kernels.py c3kmv c3onehash > gpurun_out/time_k.log 2>&1
tail -15 gpurun_out/t_k.log; cat gpurun_out/time_k.log
