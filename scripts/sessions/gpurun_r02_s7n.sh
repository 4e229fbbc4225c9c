# final c5 capture (hybrid slot layout) and launch list of the bench command
set -x
c=c5
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:tc_bloom -s 1 -c 1 -o /tmp/$c python scripts/prof_once.py $c > gpurun_out/ncu_s7n_$c.log 2>&1
ncu -i /tmp/$c.ncu-rep --page details > gpurun_out/r02e_ncu_$c.txt 2>&1
ncu -i /tmp/$c.ncu-rep --page raw --csv > gpurun_out/r02e_ncu_${c}_raw.csv 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02e_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-busy --no-secondary > gpurun_out/ncu_launch_s7n.log 2>&1
