set -x
timeout 900 python -m pytest tests/test_gpu_kmv_merge.py -x -q > gpurun_out/s5l_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5l_pytest.log
tail -5 gpurun_out/s5l_pytest.log
for v in 0 1 2 3; do
PG_TMERGE_VARIANT=$v timeout 600 python scripts/time_kernels.py c3kmv >> gpurun_out/s5l_kern.log 2>&1
done
PG_TMERGE_WARPS=12 timeout 600 python scripts/time_kernels.py c3kmv >> gpurun_out/s5l_kern.log 2>&1
PG_KMV_PARTITION=0 timeout 600 python scripts/time_kernels.py c3kmv >> gpurun_out/s5l_kern.log 2>&1
cat gpurun_out/s5l_kern.log
