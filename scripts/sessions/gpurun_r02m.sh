set -x
for v in default nofilter default; do
  if [ $v = default ]; then unset PG_LIB_PATH; else export PG_LIB_PATH=$PWD/paper_2208_11469_b200/_lib/$v/libprobgraph_b200.so; fi
  echo "== $v" >> gpurun_out/ab_m.log
  timeout 300 python scripts/time_kernels.py c3onehash >> gpurun_out/ab_m.log 2>&1
done
unset PG_LIB_PATH
timeout 600 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py tests/test_gpu_onehash_block.py -q -x > gpurun_out/t_m.log 2>&1; echo rc=$? >> gpurun_out/t_m.log
for cfg in c4:jaccard_khash c3onehash:onehash_block; do
  c=${cfg%%:*}; k=${cfg##*:}
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o /tmp/$c python scripts/prof_once.py $c > gpurun_out/ncu_m_$c.log 2>&1
  ncu -i /tmp/$c.ncu-rep --page details > gpurun_out/r02m_ncu_$c.txt 2>&1
  ncu -i /tmp/$c.ncu-rep --page raw --csv > gpurun_out/r02m_ncu_${c}_raw.csv 2>&1
done
tail -3 gpurun_out/t_m.log; cat gpurun_out/ab_m.log
