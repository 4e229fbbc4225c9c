set -x
L=paper_2208_11469_b200/_lib
for i in 1 2; do
echo "default" >> gpurun_out/s5u_kern.log
timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5u_kern.log
echo "st3" >> gpurun_out/s5u_kern.log
PG_LIB_PATH=$PWD/$L/st3/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5u_kern.log
done
PG_LIB_PATH=$PWD/$L/st3/libprobgraph_b200.so timeout 900 python -m pytest tests/test_gpu_kmv_merge.py -x -q 2>&1 | tail -3
cat gpurun_out/s5u_kern.log
