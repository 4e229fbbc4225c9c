set -x
for c in 0 1 0 1; do PG_TC_CSA=$c timeout 300 python scripts/probe_tc.py c2 id >> gpurun_out/ab_am.log 2>&1; done
for c in 0 1; do PG_TC_CSA=$c timeout 300 python scripts/time_kernels.py c4 >> gpurun_out/ab_am.log 2>&1; done
cat gpurun_out/ab_am.log
