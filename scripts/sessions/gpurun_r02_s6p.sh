set -x
L=paper_2208_11469_b200/_lib
for i in 1 2; do
for v in default l2h1 l2h2; do
echo "$v" >> gpurun_out/s6p_kern.log
if [ $v = default ]; then timeout 600 python scripts/time_kernels.py c5 2>&1 | tail -1 >> gpurun_out/s6p_kern.log
else PG_LIB_PATH=$PWD/$L/$v/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c5 2>&1 | tail -1 >> gpurun_out/s6p_kern.log; fi
done; done
cat gpurun_out/s6p_kern.log
