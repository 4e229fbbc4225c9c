set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python bench.py > gpurun_out/bench_o.json 2> gpurun_out/bench_o.err; echo rc=$? >> gpurun_out/bench_o.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_o.json 2> gpurun_out/bench_ref_o.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02o_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-busy --no-secondary > gpurun_out/ncu_launch_o.log 2>&1
tail -3 gpurun_out/bench_o.err
