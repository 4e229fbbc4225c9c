set -x
timeout 900 python -m pytest tests/test_gpu_onehash_rank.py -x -q 2>&1 | tail -3
timeout 600 python scripts/time_layout_c3.py 2>&1 | grep "onehash 1"
timeout 600 python scripts/time_kernels.py c3onehash 2>&1 | tail -1
