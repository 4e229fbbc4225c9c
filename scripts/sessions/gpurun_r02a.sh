set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_bloom_odd.py tests/test_gpu_hub.py tests/test_gpu_bench_multi.py tests/test_gpu_plugin_boundary.py -x -q > gpurun_out/t_new.log 2>&1; echo rc=$? >> gpurun_out/t_new.log
for t in 512 640 768; do for c in 0 1; do PG_HUB_THREADS=$t PG_HUB_CSA=$c timeout 300 python scripts/probe_hub.py 24 >> gpurun_out/probe_hub.log 2>&1; done; done
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 900 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo rc=$? >> gpurun_out/bench1.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench1_ref.json 2> gpurun_out/bench1_ref.err
nproc; free -g
