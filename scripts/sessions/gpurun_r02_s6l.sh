set -x
timeout 900 python -m pytest tests/test_gpu_onehash_rank.py tests/test_gpu_onehash_block.py tests/test_gpu_random_tc.py tests/test_gpu_large.py -x -q 2>&1 | tail -3
timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1
PG_ONEHASH_ROWS=id timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1
