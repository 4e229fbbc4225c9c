# round 2: full GPU tests, c5 bench (+ reference arm), launch list, ncu --set full of every config's estimator kernel
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-busy --no-secondary > gpurun_out/ncu_launch.log 2>&1
for cfg in c5:tc_bloom c4:jaccard_khash c3onehash:onehash c3kmv:kmv_ranked; do
  c=${cfg%%:*}; k=${cfg##*:}
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o /tmp/$c python scripts/prof_once.py $c > gpurun_out/ncu_$c.log 2>&1
  ncu -i /tmp/$c.ncu-rep --page details > gpurun_out/r02_ncu_$c.txt 2>&1
  ncu -i /tmp/$c.ncu-rep --page raw --csv > gpurun_out/r02_ncu_${c}_raw.csv 2>&1
  ncu -i /tmp/$c.ncu-rep --page source --csv > gpurun_out/r02_ncu_${c}_source.csv 2>&1
done
ls -la gpurun_out
