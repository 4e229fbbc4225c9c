set -x
timeout 600 python scripts/time_e2e_c5.py 20 > gpurun_out/e2e_u.log 2>&1
PG_REPO=$PWD/_r1 timeout 600 python scripts/time_e2e_c5.py 20 >> gpurun_out/e2e_u.log 2>&1
cat gpurun_out/e2e_u.log
