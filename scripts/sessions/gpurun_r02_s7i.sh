set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "clique or c5b or 4" 2>&1 | tail -2
timeout 600 python scripts/time_kernels.py c5b_bloom 2>&1 | tail -1
timeout 600 python scripts/time_kernels.py c5b_bloom 2>&1 | tail -1
