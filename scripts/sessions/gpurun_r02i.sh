set -x
for mb in 2 3 4; do PG_TC_MINB=$mb timeout 300 python scripts/probe_tc.py c5 degree >> gpurun_out/ab_i.log 2>&1; done
PG_TC_HUB=1 timeout 300 python scripts/probe_tc.py c5 degree >> gpurun_out/ab_i.log 2>&1
PG_TC_HUB=1 PG_HUB_CSA=0 timeout 300 python scripts/probe_tc.py c5 degree >> gpurun_out/ab_i.log 2>&1
PG_TC_VCACHE=0 timeout 300 python scripts/probe_tc.py c5 degree >> gpurun_out/ab_i.log 2>&1
cat gpurun_out/ab_i.log
