set -x
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t_aj.log 2>&1; echo rc=$? >> gpurun_out/t_aj.log
tail -25 gpurun_out/t_aj.log | grep -E "passed|failed|Error|assert|rc="
