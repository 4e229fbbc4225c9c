# A/B of the wide engine: default (IMAD adds, 4 CSAs) / noimad / csa3
set -x
for v in default noimad csa3 default csa3; do
  if [ $v = default ]; then unset PG_LIB_PATH; else export PG_LIB_PATH=$PWD/paper_2208_11469_b200/_lib/$v/libprobgraph_b200.so; fi
  echo "== $v" >> gpurun_out/ab_g.log
  timeout 300 python scripts/probe_tc.py c5 degree >> gpurun_out/ab_g.log 2>&1
  timeout 300 python scripts/probe_tc.py c2 id >> gpurun_out/ab_g.log 2>&1
done
unset PG_LIB_PATH
timeout 300 python scripts/time_kernels.py c4 >> gpurun_out/ab_g.log 2>&1
cat gpurun_out/ab_g.log
