set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_clique_sketch.py tests/test_gpu_large.py tests/test_gpu_parity.py -q -x > gpurun_out/t_d.log 2>&1; echo rc=$? >> gpurun_out/t_d.log
for o in degree id; do PG_TC_ORIENT=$o timeout 300 python scripts/time_kernels.py c4 >> gpurun_out/time_d.log 2>&1; done
timeout 600 python scripts/time_kernels.py c5b_bloom c5b_khash c5b_onehash c5b_kmv >> gpurun_out/time_d.log 2>&1
PG_K=32 timeout 600 python scripts/time_kernels.py c5b_khash >> gpurun_out/time_d.log 2>&1
cat gpurun_out/time_d.log
