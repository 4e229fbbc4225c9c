set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/t_ba.log 2>&1; echo rc=$? >> gpurun_out/t_ba.log
tail -3 gpurun_out/t_ba.log
timeout 900 python bench.py > gpurun_out/bench_ba.json 2> gpurun_out/bench_ba.err; echo rc=$?
tail -c 3000 gpurun_out/bench_ba.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_ba.json 2> gpurun_out/bench_ref_ba.err; echo rc=$?
tail -c 1500 gpurun_out/bench_ref_ba.json
