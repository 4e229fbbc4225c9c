set -x
c=c3kmv
PG_TMERGE_VARIANT=1 timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:kmv_tmerge -s 1 -c 1 -o /tmp/$c python scripts/prof_once.py $c > gpurun_out/ncu_s5m_$c.log 2>&1
ncu -i /tmp/$c.ncu-rep --page details > gpurun_out/s5m_ncu_$c.txt 2>&1
ncu -i /tmp/$c.ncu-rep --page raw --csv > gpurun_out/s5m_ncu_${c}_raw.csv 2>&1
ncu -i /tmp/$c.ncu-rep --page source --csv > gpurun_out/s5m_ncu_${c}_src.csv 2>&1
ls -la gpurun_out/s5m_*
