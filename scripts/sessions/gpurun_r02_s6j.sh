set -x
c=c3onehash
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:onehash_block -s 1 -c 1 -o /tmp/$c python scripts/prof_once.py $c > gpurun_out/ncu_s6j_$c.log 2>&1
ncu -i /tmp/$c.ncu-rep --page source --csv > gpurun_out/s6j_ncu_${c}_src.csv 2>&1
