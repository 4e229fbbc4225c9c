set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5a_pytest.log
tail -3 gpurun_out/s5a_pytest.log
timeout 900 python bench.py > gpurun_out/s5a_bench.json 2> gpurun_out/s5a_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/s5a_bench.json
timeout 600 python scripts/time_kernels.py c3onehash c3kmv c4 c5 > gpurun_out/s5a_kern.log 2>&1
cat gpurun_out/s5a_kern.log
