set -x
timeout 600 python scripts/time_layout_c3.py 2>&1 | tail -24
