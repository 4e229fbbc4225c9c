set -x
for c in -1 0 10 25 50; do
  if [ $c = -1 ]; then unset PG_TC_CARVEOUT; else export PG_TC_CARVEOUT=$c; fi
  timeout 300 python scripts/probe_tc.py c5 degree >> gpurun_out/ab_s.log 2>&1
done
cat gpurun_out/ab_s.log
