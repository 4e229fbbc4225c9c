set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s6i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s6i_pytest.log
tail -3 gpurun_out/s6i_pytest.log
timeout 600 python scripts/time_kernels.py c3onehash c3kmv 2>&1 | tail -2
