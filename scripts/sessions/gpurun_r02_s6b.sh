set -x
L=paper_2208_11469_b200/_lib
for i in 1 2; do
for v in r1 default r4; do
echo "$v" >> gpurun_out/s6b_kern.log
if [ $v = default ]; then timeout 600 python scripts/time_kernels.py c5b_bloom 2>&1 | tail -1 >> gpurun_out/s6b_kern.log
else PG_LIB_PATH=$PWD/$L/$v/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c5b_bloom 2>&1 | tail -1 >> gpurun_out/s6b_kern.log; fi
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "clique or c5b or 4" 2>&1 | tail -3
cat gpurun_out/s6b_kern.log
