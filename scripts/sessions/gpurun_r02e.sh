set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_clique_sketch.py -q -x > gpurun_out/t_e.log 2>&1; echo rc=$? >> gpurun_out/t_e.log
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x >> gpurun_out/t_e.log 2>&1; echo rc=$? >> gpurun_out/t_e.log
timeout 600 python scripts/time_kernels.py c5b_khash c5b_onehash c5b_kmv > gpurun_out/time_e.log 2>&1
tail -5 gpurun_out/t_e.log; cat gpurun_out/time_e.log
