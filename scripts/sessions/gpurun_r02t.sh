set -x
timeout 600 python scripts/time_e2e_c5.py 20 > gpurun_out/e2e_t.log 2>&1
PG_TC_ORIENT=id timeout 600 python scripts/time_e2e_c5.py 20 >> gpurun_out/e2e_t.log 2>&1
cat gpurun_out/e2e_t.log
