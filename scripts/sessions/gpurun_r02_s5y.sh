set -x
L=paper_2208_11469_b200/_lib
for i in 1 2 3; do
echo "new" >> gpurun_out/s5y_kern.log
timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5y_kern.log
echo "old (fixed chunk)" >> gpurun_out/s5y_kern.log
PG_LIB_PATH=$PWD/$L/oldchunk/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5y_kern.log
done
cat gpurun_out/s5y_kern.log
