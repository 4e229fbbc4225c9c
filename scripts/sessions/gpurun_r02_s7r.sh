set -x
timeout 900 python -m pytest tests/test_gpu_hybrid_layout.py tests/test_gpu_large.py -x -q 2>&1 | tail -2
timeout 900 python scripts/time_shards.py c5 2>&1 | tail -1
timeout 600 python scripts/time_kernels.py c5 2>&1 | tail -1
