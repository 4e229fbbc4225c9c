# final-state run: GPU tests, default bench, launch list of the bench command
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5x_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5x_pytest.log
tail -3 gpurun_out/s5x_pytest.log
timeout 900 python bench.py > gpurun_out/s5x_bench.json 2> gpurun_out/s5x_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s5x_bench_ref.json 2> gpurun_out/s5x_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02d_launches_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-busy --no-secondary > gpurun_out/ncu_launch_s5x.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
