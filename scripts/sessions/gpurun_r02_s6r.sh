set -x
L=paper_2208_11469_b200/_lib
echo "default" >> gpurun_out/s6r_kern.log
timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1 >> gpurun_out/s6r_kern.log
echo "per-lane 16" >> gpurun_out/s6r_kern.log
PG_LIB_PATH=$PWD/$L/pl16/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1 >> gpurun_out/s6r_kern.log
cat gpurun_out/s6r_kern.log
