set -x
for r in _b_eec858b _b_5741076; do
  echo "== $r" >> gpurun_out/prof_y.log
  PG_REPO=$PWD/$r timeout 600 python scripts/prof_e2e_host.py 2>&1 | head -22 >> gpurun_out/prof_y.log
done
cat gpurun_out/prof_y.log
