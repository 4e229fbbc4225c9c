set -x
timeout 900 python -m pytest tests/test_gpu_generic.py tests/test_gpu_guards.py -q -x > gpurun_out/t_ad.log 2>&1; echo rc=$? >> gpurun_out/t_ad.log
timeout 600 python scripts/time_e2e_c5.py 20 > gpurun_out/e2e_ad.log 2>&1
timeout 600 python scripts/time_e2e_c5.py 24 >> gpurun_out/e2e_ad.log 2>&1
tail -3 gpurun_out/t_ad.log; cat gpurun_out/e2e_ad.log
