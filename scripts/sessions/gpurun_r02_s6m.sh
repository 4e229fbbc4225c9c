# final-state run: GPU tests, default bench + reference arm, smoke
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s6m_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s6m_pytest.log
tail -3 gpurun_out/s6m_pytest.log
timeout 900 python bench.py > gpurun_out/s6m_bench.json 2> gpurun_out/s6m_bench.err; echo "bench rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
