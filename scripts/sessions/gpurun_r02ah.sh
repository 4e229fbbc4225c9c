set -x
timeout 900 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_plugin_boundary.py tests/test_gpu_parity.py tests/test_gpu_clique_sketch.py -q -x > gpurun_out/t_ah.log 2>&1; echo rc=$? >> gpurun_out/t_ah.log
timeout 300 python scripts/time_scalar.py > gpurun_out/scalar_ah.log 2>&1
tail -3 gpurun_out/t_ah.log; cat gpurun_out/scalar_ah.log
