set -x
L=paper_2208_11469_b200/_lib
for v in base unc rev s2 s2v; do
echo "alt $v" >> gpurun_out/s5p_kern.log
PG_LIB_PATH=$PWD/$L/$v/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5p_kern.log
done
echo "default" >> gpurun_out/s5p_kern.log
timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5p_kern.log
echo "default carve 70 / variant1" >> gpurun_out/s5p_kern.log
PG_TMERGE_CARVEOUT=70 timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5p_kern.log
PG_TMERGE_VARIANT=1 timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5p_kern.log
timeout 900 python -m pytest tests/test_gpu_kmv_merge.py -x -q 2>&1 | tail -3
PG_LIB_PATH=$PWD/$L/s2v/libprobgraph_b200.so timeout 900 python -m pytest tests/test_gpu_kmv_merge.py -x -q 2>&1 | tail -3
cat gpurun_out/s5p_kern.log
