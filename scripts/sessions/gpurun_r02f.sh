# A/B of the wide engine: default (xor reduce + IMAD adds) / noimad / old
set -x
for v in default noimad old default; do
  if [ $v = default ]; then unset PG_LIB_PATH; else export PG_LIB_PATH=$PWD/paper_2208_11469_b200/_lib/$v/libprobgraph_b200.so; fi
  echo "== $v" >> gpurun_out/ab_f.log
  timeout 300 python scripts/probe_tc.py c5 degree >> gpurun_out/ab_f.log 2>&1
  timeout 300 python scripts/probe_tc.py c2 id >> gpurun_out/ab_f.log 2>&1
  timeout 300 python scripts/time_kernels.py c4 >> gpurun_out/ab_f.log 2>&1
done
unset PG_LIB_PATH
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_hub.py -q -x > gpurun_out/t_f.log 2>&1; echo rc=$? >> gpurun_out/t_f.log
tail -3 gpurun_out/t_f.log; cat gpurun_out/ab_f.log
