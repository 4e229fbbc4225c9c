set -x
L=paper_2208_11469_b200/_lib
for i in 1 2; do
echo "default" >> gpurun_out/s5z_kern.log
timeout 600 python scripts/time_kernels.py c5 2>&1 | tail -1 >> gpurun_out/s5z_kern.log
for v in ust1 ust2; do
echo "$v" >> gpurun_out/s5z_kern.log
PG_LIB_PATH=$PWD/$L/$v/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c5 2>&1 | tail -1 >> gpurun_out/s5z_kern.log
done
done
cat gpurun_out/s5z_kern.log
