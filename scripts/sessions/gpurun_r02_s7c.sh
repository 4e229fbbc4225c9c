set -x
timeout 900 python -m pytest tests/test_gpu_clique_sketch.py tests/test_gpu_determinism.py tests/test_gpu_guards.py tests/test_gpu_generic.py -x -q 2>&1 | tail -3
timeout 900 python scripts/time_kernels.py c5b_khash c5b_onehash c5b_kmv 2>&1 | tail -3
