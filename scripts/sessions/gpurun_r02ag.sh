set -x
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:kmv_hash -s 1 -c 1 -o /tmp/kh python scripts/prof_once.py c3kmv > gpurun_out/ncu_ag.log 2>&1
ncu -i /tmp/kh.ncu-rep --page raw --csv > gpurun_out/r02ag_kmvhash_raw.csv 2>&1
ncu -i /tmp/kh.ncu-rep --page source --csv > gpurun_out/r02ag_kmvhash_source.csv 2>&1
ncu -i /tmp/kh.ncu-rep --page details > gpurun_out/r02ag_kmvhash.txt 2>&1
tail -3 gpurun_out/ncu_ag.log
