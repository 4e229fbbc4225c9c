set -x
timeout 900 python bench.py > gpurun_out/s6f_bench.json 2> gpurun_out/s6f_bench.err; echo "bench rc=$?"
