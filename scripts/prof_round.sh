set -x
[ -n "$SKIP_BENCH" ] || python bench.py > gpurun_out/bench_r01d.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r01d_launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-busy --no-secondary > gpurun_out/ncu_launch.log 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:tc_bloom_wide -s 3 -c 1 -o /tmp/tc python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-busy --no-secondary > gpurun_out/ncu_tc.log 2>&1
ncu -i /tmp/tc.ncu-rep --page details > gpurun_out/r01d_ncu_tc_c2.txt 2>&1
ncu -i /tmp/tc.ncu-rep --page raw --csv > gpurun_out/r01d_ncu_tc_c2_raw.csv 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:kmv_ranked -s 1 -c 1 -o /tmp/kmv python scripts/prof_sorted_once.py kmv > gpurun_out/ncu_kmv.log 2>&1
ncu -i /tmp/kmv.ncu-rep --page details > gpurun_out/r01d_ncu_kmv_ranked_s20.txt 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:onehash_block -s 1 -c 1 -o /tmp/oh python scripts/prof_sorted_once.py onehash > gpurun_out/ncu_oh.log 2>&1
ncu -i /tmp/oh.ncu-rep --page details > gpurun_out/r01d_ncu_onehash_block_s20.txt 2>&1
ls -la gpurun_out
