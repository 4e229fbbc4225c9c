set -x
export PG_TMERGE_VARIANT=1
for c in 100 75 60 50; do
echo "carveout $c" >> gpurun_out/s5n_kern.log
PG_TMERGE_CARVEOUT=$c timeout 600 python scripts/time_kernels.py c3kmv >> gpurun_out/s5n_kern.log 2>&1
done
echo "id orient carve 100 / 60" >> gpurun_out/s5n_kern.log
PG_TC_ORIENT=id PG_TMERGE_CARVEOUT=100 timeout 600 python scripts/time_kernels.py c3kmv >> gpurun_out/s5n_kern.log 2>&1
PG_TC_ORIENT=id PG_TMERGE_CARVEOUT=60 timeout 600 python scripts/time_kernels.py c3kmv >> gpurun_out/s5n_kern.log 2>&1
echo "warps 8 carve 50" >> gpurun_out/s5n_kern.log
PG_TMERGE_WARPS=8 PG_TMERGE_CARVEOUT=50 timeout 600 python scripts/time_kernels.py c3kmv >> gpurun_out/s5n_kern.log 2>&1
cat gpurun_out/s5n_kern.log
