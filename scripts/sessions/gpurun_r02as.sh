set -x
for v in default kmvp4 kmvp4m4; do
  if [ $v = default ]; then unset PG_LIB_PATH; else export PG_LIB_PATH=$PWD/paper_2208_11469_b200/_lib/$v/libprobgraph_b200.so; fi
  echo "== $v" >> gpurun_out/ab_as.log
  timeout 300 python scripts/time_kernels.py c3kmv >> gpurun_out/ab_as.log 2>&1
done
export PG_LIB_PATH=$PWD/paper_2208_11469_b200/_lib/kmvp4/libprobgraph_b200.so
timeout 600 python -m pytest tests/test_gpu_kmv_ranked.py -q -x > gpurun_out/t_as.log 2>&1; echo rc=$? >> gpurun_out/t_as.log
cat gpurun_out/ab_as.log; tail -2 gpurun_out/t_as.log
