set -x
timeout 900 python -m pytest tests/test_gpu_hybrid_layout.py tests/test_gpu_large.py tests/test_gpu_hub.py tests/test_gpu_sharded.py tests/test_gpu_bench_multi.py -x -q 2>&1 | tail -2
timeout 900 python scripts/time_shards.py c5 2>&1 | tail -1
bash scripts/sessions/gpurun_r02_s7n.sh
