set -x
timeout 900 python scripts/fuzz_engines.py 240 2>&1 | tail -5
