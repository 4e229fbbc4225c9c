set -x
timeout 900 python -m pytest tests/test_gpu_generic.py -q -x > gpurun_out/t_l.log 2>&1; echo rc=$? >> gpurun_out/t_l.log
timeout 1200 python -m pytest tests -q -m gpu -x >> gpurun_out/t_l.log 2>&1; echo rc=$? >> gpurun_out/t_l.log
grep -E "passed|failed|rc=|Error|assert" gpurun_out/t_l.log | tail -30
