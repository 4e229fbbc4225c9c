set -x
timeout 900 python -m pytest tests/test_gpu_kmv_merge.py tests/test_gpu_kmv_ranked.py -x -q > gpurun_out/s5b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5b_pytest.log
tail -15 gpurun_out/s5b_pytest.log
timeout 600 python scripts/time_kernels.py c3kmv > gpurun_out/s5b_kern.log 2>&1
PG_KMV_PARTITION=0 timeout 600 python scripts/time_kernels.py c3kmv >> gpurun_out/s5b_kern.log 2>&1
PG_TC_ORIENT=id timeout 600 python scripts/time_kernels.py c3kmv >> gpurun_out/s5b_kern.log 2>&1
PG_TMERGE_WARPS=8 timeout 600 python scripts/time_kernels.py c3kmv >> gpurun_out/s5b_kern.log 2>&1
PG_KMV_ENGINE=ranked timeout 600 python scripts/time_kernels.py c3kmv >> gpurun_out/s5b_kern.log 2>&1
cat gpurun_out/s5b_kern.log
