set -x
L=paper_2208_11469_b200/_lib
echo "default" >> gpurun_out/s5r_kern.log
timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5r_kern.log
for v in st2; do
echo "alt $v" >> gpurun_out/s5r_kern.log
PG_LIB_PATH=$PWD/$L/$v/libprobgraph_b200.so timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5r_kern.log
done
echo "carve 80, warps 18, warps 16" >> gpurun_out/s5r_kern.log
PG_TMERGE_CARVEOUT=80 timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5r_kern.log
PG_TMERGE_WARPS=18 timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5r_kern.log
PG_TMERGE_WARPS=16 timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s5r_kern.log
cat gpurun_out/s5r_kern.log
c=c3kmv
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:kmv_tmerge -s 1 -c 1 -o /tmp/$c python scripts/prof_once.py $c > gpurun_out/ncu_s5r_$c.log 2>&1
ncu -i /tmp/$c.ncu-rep --page details > gpurun_out/s5r_ncu_$c.txt 2>&1
ncu -i /tmp/$c.ncu-rep --page raw --csv > gpurun_out/s5r_ncu_${c}_raw.csv 2>&1
ncu -i /tmp/$c.ncu-rep --page source --csv > gpurun_out/s5r_ncu_${c}_src.csv 2>&1
