set -x
c=c5b
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:clique4_bloom -s 1 -c 1 -o /tmp/$c python scripts/prof_c5b.py > gpurun_out/ncu_s7h_$c.log 2>&1
ncu -i /tmp/$c.ncu-rep --page details > gpurun_out/r02e_ncu_$c.txt 2>&1
ncu -i /tmp/$c.ncu-rep --page source --csv > gpurun_out/s7h_ncu_${c}_src.csv 2>&1
