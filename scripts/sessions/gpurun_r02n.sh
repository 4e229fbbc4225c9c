set -x
for v in default kh5 kh6 default; do
  if [ $v = default ]; then unset PG_LIB_PATH; else export PG_LIB_PATH=$PWD/paper_2208_11469_b200/_lib/$v/libprobgraph_b200.so; fi
  echo "== $v" >> gpurun_out/ab_n.log
  timeout 300 python scripts/time_kernels.py c4 >> gpurun_out/ab_n.log 2>&1
done
cat gpurun_out/ab_n.log
