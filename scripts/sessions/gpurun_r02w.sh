set -x
for r in . _b_eec858b _b_1e2d429 _b_4b52a2a _r1 .; do
  echo "== $r" >> gpurun_out/e2e_w.log
  PG_REPO=$PWD/$r timeout 600 python scripts/time_e2e_c5.py 20 >> gpurun_out/e2e_w.log 2>&1
done
cat gpurun_out/e2e_w.log
