# compute-sanitizer over scripts/sanitize_cases.py (every kernel family once)
set -x
timeout 300 python scripts/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo rc=$? >> gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1; echo rc=$? >> gpurun_out/san_$tool.log
done
tail -4 gpurun_out/san_*.log
