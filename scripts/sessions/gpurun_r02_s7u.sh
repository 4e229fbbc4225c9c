set -x
timeout 900 python -m pytest tests/test_gpu_hybrid_layout.py -x -q 2>&1 | tail -2
bash scripts/sessions/gpurun_r02_s7j.sh
