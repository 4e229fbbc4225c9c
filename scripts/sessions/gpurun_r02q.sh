set -x
for v in default sub4m4 sub4m5 sub2m5 default; do
  if [ $v = default ]; then unset PG_LIB_PATH; else export PG_LIB_PATH=$PWD/paper_2208_11469_b200/_lib/$v/libprobgraph_b200.so; fi
  echo "== $v" >> gpurun_out/ab_q.log
  timeout 300 python scripts/probe_tc.py c5 degree >> gpurun_out/ab_q.log 2>&1
done
cat gpurun_out/ab_q.log
