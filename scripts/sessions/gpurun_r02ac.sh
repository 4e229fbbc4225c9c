set -x
for v in noseg default noseg; do
  if [ $v = default ]; then unset PG_LIB_PATH; else export PG_LIB_PATH=$PWD/paper_2208_11469_b200/_lib/$v/libprobgraph_b200.so; fi
  echo "== $v" >> gpurun_out/e2e_ac.log
  timeout 600 python scripts/time_e2e_c5.py 20 >> gpurun_out/e2e_ac.log 2>&1
done
cat gpurun_out/e2e_ac.log
