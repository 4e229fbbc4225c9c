set -x
timeout 900 python -m pytest tests/test_gpu_clique_sketch.py tests/test_gpu_generic.py tests/test_gpu_guards.py -q -x > gpurun_out/t_p.log 2>&1; echo rc=$? >> gpurun_out/t_p.log
timeout 600 python scripts/time_kernels.py c5b_khash c5b_onehash c5b_kmv > gpurun_out/time_p.log 2>&1
tail -3 gpurun_out/t_p.log; cat gpurun_out/time_p.log
