set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5s_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5s_pytest.log
tail -4 gpurun_out/s5s_pytest.log
timeout 900 python bench.py > gpurun_out/s5s_bench.json 2> gpurun_out/s5s_bench.err; echo "bench rc=$?"
