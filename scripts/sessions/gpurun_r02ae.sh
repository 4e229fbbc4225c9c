set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t_ae.log 2>&1; echo rc=$? >> gpurun_out/t_ae.log
timeout 1200 python bench.py > gpurun_out/bench_ae.json 2> gpurun_out/bench_ae.err; echo rc=$? >> gpurun_out/bench_ae.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_ae.json 2> gpurun_out/bench_ref_ae.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ae.log 2>&1; echo rc=$? >> gpurun_out/smoke_ae.log
tail -3 gpurun_out/t_ae.log; tail -2 gpurun_out/bench_ae.err; cat gpurun_out/smoke_ae.log
