set -x
L=paper_2208_11469_b200/_lib
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_sharded.py tests/test_gpu_generic.py -x -q -k "clique or c5b or 4" 2>&1 | tail -3
for i in 1 2; do
echo "dynamic" >> gpurun_out/s7a_kern.log
timeout 600 python scripts/time_kernels.py c5b_bloom 2>&1 | tail -1 >> gpurun_out/s7a_kern.log
echo "static" >> gpurun_out/s7a_kern.log
PG_LIB_PATH=$PWD/$L/c4static/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c5b_bloom 2>&1 | tail -1 >> gpurun_out/s7a_kern.log
done
cat gpurun_out/s7a_kern.log
