set -x
timeout 900 python -m pytest tests/test_gpu_kmv_merge.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -3
for b in 8 4 1; do
echo "buckets $b" >> gpurun_out/s6o_kern.log
PG_KMV_BUCKETS=$b timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s6o_kern.log
done
cat gpurun_out/s6o_kern.log
