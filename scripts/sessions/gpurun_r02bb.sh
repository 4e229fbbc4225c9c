set -x
L=$PWD/paper_2208_11469_b200/_lib
for rep in 1 2; do
for v in default oldtr; do
  if [ $v = default ]; then unset PG_LIB_PATH; else export PG_LIB_PATH=$L/$v/libprobgraph_b200.so; fi
  echo "== $v" >> gpurun_out/ab_bb.log
  timeout 300 python scripts/time_kernels.py c5 c2 c4 >> gpurun_out/ab_bb.log 2>&1
done
done
unset PG_LIB_PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_guards.py tests/test_gpu_determinism.py -q -x -m gpu > gpurun_out/t_bb.log 2>&1; echo rc=$? >> gpurun_out/t_bb.log
cat gpurun_out/ab_bb.log; tail -3 gpurun_out/t_bb.log
