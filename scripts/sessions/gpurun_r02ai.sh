set -x
timeout 600 python -m pytest tests/test_gpu_with_set.py tests/test_gpu_plugin_boundary.py tests/test_gpu_parity.py -q -x > gpurun_out/t_ai.log 2>&1; echo rc=$? >> gpurun_out/t_ai.log
timeout 300 python scripts/time_scalar.py > gpurun_out/scalar_ai.log 2>&1
tail -30 gpurun_out/t_ai.log | grep -E "passed|failed|Error|assert|rc=" ; cat gpurun_out/scalar_ai.log
