set -x
timeout 900 python -m pytest tests/test_gpu_onehash_rank.py tests/test_gpu_onehash_block.py tests/test_gpu_random_tc.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -5
for i in 1 2; do
for cfgv in "degree sorted" "id sorted" "degree plain"; do
set -- $cfgv
echo "orient $1 layout $2" >> gpurun_out/s6d_kern.log
PG_TC_ORIENT=$1 PG_ONEHASH_LAYOUT=$2 timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1 >> gpurun_out/s6d_kern.log
done; done
cat gpurun_out/s6d_kern.log
