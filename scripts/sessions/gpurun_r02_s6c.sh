set -x
timeout 900 python -m pytest tests/test_gpu_onehash_rank.py tests/test_gpu_onehash_block.py tests/test_gpu_random_tc.py -x -q 2>&1 | tail -5
for i in 1 2; do
echo "rank rows" >> gpurun_out/s6c_kern.log
timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1 >> gpurun_out/s6c_kern.log
echo "id rows" >> gpurun_out/s6c_kern.log
PG_ONEHASH_ROWS=id timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1 >> gpurun_out/s6c_kern.log
done
cat gpurun_out/s6c_kern.log
