set -x
L=paper_2208_11469_b200/_lib
for c in 2 4 16 32; do
echo "chunk $c" >> gpurun_out/s7b_kern.log
PG_LIB_PATH=$PWD/$L/c4c$c/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c5b_bloom 2>&1 | tail -1 >> gpurun_out/s7b_kern.log
done
cat gpurun_out/s7b_kern.log
