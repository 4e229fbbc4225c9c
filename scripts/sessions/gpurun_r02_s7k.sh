set -x
timeout 900 python -m pytest tests/test_gpu_hybrid_layout.py tests/test_gpu_large.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_bench_multi.py -x -q 2>&1 | tail -3
PG_TC_HYBRID=3 timeout 600 python scripts/time_kernels.py c5 2>&1 | tail -1
timeout 600 python scripts/time_layout.py 2>&1 | tail -6
