# final captures of the two c3 kernels
set -x
for cfg in c3onehash:onehash_block c3kmv:kmv_tmerge; do
  c=${cfg%%:*}; k=${cfg##*:}
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o /tmp/$c python scripts/prof_once.py $c > gpurun_out/ncu_s6s_$c.log 2>&1
  ncu -i /tmp/$c.ncu-rep --page details > gpurun_out/r02e_ncu_$c.txt 2>&1
  ncu -i /tmp/$c.ncu-rep --page raw --csv > gpurun_out/r02e_ncu_${c}_raw.csv 2>&1
done
