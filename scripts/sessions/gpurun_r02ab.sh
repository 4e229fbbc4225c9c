set -x
echo "== default env=${CUDA_MODULE_LOADING}" >> gpurun_out/e2e_ab.log
timeout 600 python scripts/time_e2e_c5.py 20 >> gpurun_out/e2e_ab.log 2>&1
echo "== default EAGER" >> gpurun_out/e2e_ab.log
CUDA_MODULE_LOADING=EAGER timeout 600 python scripts/time_e2e_c5.py 20 >> gpurun_out/e2e_ab.log 2>&1
echo "== default LAZY" >> gpurun_out/e2e_ab.log
CUDA_MODULE_LOADING=LAZY timeout 600 python scripts/time_e2e_c5.py 20 >> gpurun_out/e2e_ab.log 2>&1
echo "== nogen EAGER" >> gpurun_out/e2e_ab.log
CUDA_MODULE_LOADING=EAGER PG_LIB_PATH=$PWD/paper_2208_11469_b200/_lib/nogen/libprobgraph_b200.so timeout 600 python scripts/time_e2e_c5.py 20 >> gpurun_out/e2e_ab.log 2>&1
cat gpurun_out/e2e_ab.log
