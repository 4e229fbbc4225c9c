set -x
L=paper_2208_11469_b200/_lib
for c in 1 2 32; do
echo "chunk $c" >> gpurun_out/s7d_kern.log
PG_LIB_PATH=$PWD/$L/c4s$c/libprobgraph_b200.so timeout 900 python scripts/time_kernels.py c5b_khash c5b_onehash c5b_kmv 2>&1 | tail -3 >> gpurun_out/s7d_kern.log
done
cat gpurun_out/s7d_kern.log
