ncu -f --set full --clock-control none -k regex:tc_bloom_wide -s 1 -c 1 -o /tmp/c5 python scripts/prof_c5_once.py > gpurun_out/ncu_c5.log 2>&1
ncu -i /tmp/c5.ncu-rep --page details > gpurun_out/r01d_ncu_tc_c5.txt 2>&1
ncu -i /tmp/c5.ncu-rep --page raw --csv > gpurun_out/r01d_ncu_tc_c5_raw.csv 2>&1
ncu -f --set full --clock-control none -k regex:jaccard_khash -s 1 -c 1 -o /tmp/c4 python scripts/prof_c4_jaccard.py > gpurun_out/ncu_c4.log 2>&1
ncu -i /tmp/c4.ncu-rep --page details > gpurun_out/r01d_ncu_jaccard_c4.txt 2>&1
ncu -i /tmp/c4.ncu-rep --page raw --csv > gpurun_out/r01d_ncu_jaccard_c4_raw.csv 2>&1
