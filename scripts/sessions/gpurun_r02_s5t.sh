set -x
L=paper_2208_11469_b200/_lib
timeout 900 python -m pytest tests/test_gpu_onehash_block.py tests/test_gpu_random_tc.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
echo "filter" >> gpurun_out/s5t_kern.log
timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1 >> gpurun_out/s5t_kern.log
echo "nofilter" >> gpurun_out/s5t_kern.log
PG_LIB_PATH=$PWD/$L/nofilt/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1 >> gpurun_out/s5t_kern.log
cat gpurun_out/s5t_kern.log
