set -x
timeout 900 python -m pytest tests/test_gpu_kmv_merge.py tests/test_gpu_sharded.py tests/test_gpu_determinism.py -x -q 2>&1 | tail -3
timeout 900 python scripts/time_shards.py c3 2>&1 | tail -3
