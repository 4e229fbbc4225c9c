set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s6e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s6e_pytest.log
tail -3 gpurun_out/s6e_pytest.log
timeout 900 python scripts/time_shards.py c3 2>&1 | tail -2
c=c3onehash
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:onehash_block -s 1 -c 1 -o /tmp/$c python scripts/prof_once.py $c > gpurun_out/ncu_s6e_$c.log 2>&1
ncu -i /tmp/$c.ncu-rep --page details > gpurun_out/s6e_ncu_$c.txt 2>&1
ncu -i /tmp/$c.ncu-rep --page raw --csv > gpurun_out/s6e_ncu_${c}_raw.csv 2>&1
