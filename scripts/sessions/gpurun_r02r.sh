set -x
timeout 1200 python -m pytest tests/test_gpu_large.py -q -rs > gpurun_out/t_r.log 2>&1; echo rc=$? >> gpurun_out/t_r.log
tail -8 gpurun_out/t_r.log
