set -x
for r in _b_eec858b . _b_eec858b .; do
  echo "== $r" >> gpurun_out/e2e_z.log
  PG_REPO=$PWD/$r timeout 600 python scripts/time_e2e_c5.py 20 >> gpurun_out/e2e_z.log 2>&1
done
cat gpurun_out/e2e_z.log
