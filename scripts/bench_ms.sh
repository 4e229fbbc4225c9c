#!/bin/bash
# ms_per_step of a short headline bench run (dev tool): scripts/bench_ms.sh TAG
python bench.py --steps 30 --no-secondary --no-cpu-baseline --e2e-steps 0 2>/dev/null | grep '^{' | python -c "import json,sys; print('$1', json.loads(sys.stdin.read())['ms_per_step'])"
