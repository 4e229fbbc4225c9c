set -x
L=paper_2208_11469_b200/_lib
for v in default ohu2 ohu4 ohu8; do
echo "$v" >> gpurun_out/s6k_kern.log
if [ $v = default ]; then timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1 >> gpurun_out/s6k_kern.log
else PG_LIB_PATH=$PWD/$L/$v/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1 >> gpurun_out/s6k_kern.log; fi
done
cat gpurun_out/s6k_kern.log
