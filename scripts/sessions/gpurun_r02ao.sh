# final-state captures: c5 headline kernel (full set + source), c4 / c3 kernels, bench launch list
set -x
for cfg in c5:tc_bloom c4:jaccard_khash c3onehash:onehash_block c3kmv:kmv_ranked; do
  c=${cfg%%:*}; k=${cfg##*:}
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o /tmp/$c python scripts/prof_once.py $c > gpurun_out/ncu_ao_$c.log 2>&1
  ncu -i /tmp/$c.ncu-rep --page details > gpurun_out/r02c_ncu_$c.txt 2>&1
  ncu -i /tmp/$c.ncu-rep --page raw --csv > gpurun_out/r02c_ncu_${c}_raw.csv 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02c_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-busy --no-secondary > gpurun_out/ncu_launch_ao.log 2>&1
ls gpurun_out/r02c_*
