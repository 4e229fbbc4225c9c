set -x
for cfg in c5 c2; do
for csa in 0 1; do for vc in 0 1; do for mb in 2 3; do
PG_TC_CSA=$csa PG_TC_VCACHE=$vc PG_TC_MINB=$mb timeout 300 python scripts/probe_tc.py $cfg >> gpurun_out/probe_tc.log 2>&1
done; done; done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__t_sector_hit_rate.pct,sm__inst_executed_pipe_xu.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.sum --clock-control none -k regex:tc_bloom_wide -s 2 -c 4 python scripts/probe_tc.py c5 id degree > gpurun_out/ncu_orient.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hub.py tests/test_gpu_random_tc.py tests/test_gpu_parity.py tests/test_gpu_bench_multi.py -x -q > gpurun_out/t_b.log 2>&1; echo rc=$? >> gpurun_out/t_b.log
timeout 900 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo rc=$? >> gpurun_out/bench2.err
