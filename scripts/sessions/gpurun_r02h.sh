set -x
for i in 1 2; do
timeout 300 python scripts/probe_tc.py c5 degree >> gpurun_out/ab_h.log 2>&1
timeout 300 python scripts/probe_tc.py c2 id >> gpurun_out/ab_h.log 2>&1
done
timeout 300 python scripts/time_kernels.py c4 >> gpurun_out/ab_h.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t_h.log 2>&1; echo rc=$? >> gpurun_out/t_h.log
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:tc_bloom -s 1 -c 1 -o /tmp/c5 python scripts/prof_once.py c5 > gpurun_out/ncu_c5h.log 2>&1
ncu -i /tmp/c5.ncu-rep --page raw --csv > gpurun_out/r02h_ncu_c5_raw.csv 2>&1
ncu -i /tmp/c5.ncu-rep --page details > gpurun_out/r02h_ncu_c5.txt 2>&1
tail -3 gpurun_out/t_h.log; cat gpurun_out/ab_h.log
