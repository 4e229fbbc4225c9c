set -x
timeout 900 python -m pytest tests/test_gpu_kmv_merge.py -x -q > gpurun_out/s5o_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5o_pytest.log
tail -5 gpurun_out/s5o_pytest.log
for v in 0 1 2; do
for c in 100 70; do
echo "variant $v carve $c" >> gpurun_out/s5o_kern.log
PG_TMERGE_CARVEOUT=$c PG_TMERGE_VARIANT=$v timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5o_kern.log
done; done
echo "nopart" >> gpurun_out/s5o_kern.log
PG_KMV_PARTITION=0 timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5o_kern.log
cat gpurun_out/s5o_kern.log
