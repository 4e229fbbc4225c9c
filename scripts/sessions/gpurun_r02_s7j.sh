set -x
for t in 2 3 4 5; do
echo "hybrid thr $t" >> gpurun_out/s7j_kern.log
PG_TC_HYBRID=$t timeout 600 python scripts/time_kernels.py c5 2>&1 | tail -1 >> gpurun_out/s7j_kern.log
done
cat gpurun_out/s7j_kern.log
