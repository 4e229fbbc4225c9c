set -x
echo new; timeout 600 python scripts/time_k_sweep.py 2>&1 | tail -6
echo old; PG_KMV_ENGINE=ranked PG_ONEHASH_ROWS=id timeout 600 python scripts/time_k_sweep.py 2>&1 | tail -6
