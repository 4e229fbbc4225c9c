set -x
for o in 0 1 0 1; do
  echo "== low_first=$o" >> gpurun_out/e2e_al.log
  PG_UPLOAD_LOW_FIRST=$o timeout 600 python scripts/time_e2e_c5.py 20 >> gpurun_out/e2e_al.log 2>&1
  PG_UPLOAD_LOW_FIRST=$o timeout 600 python scripts/time_e2e_c5.py 24 >> gpurun_out/e2e_al.log 2>&1
done
PG_UPLOAD_LOW_FIRST=1 timeout 600 python -m pytest tests/test_gpu_e2e.py -q -x > gpurun_out/t_al.log 2>&1; echo rc=$? >> gpurun_out/t_al.log
cat gpurun_out/e2e_al.log | grep -E "==|e2e"; tail -2 gpurun_out/t_al.log
