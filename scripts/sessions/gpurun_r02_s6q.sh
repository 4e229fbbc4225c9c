set -x
L=paper_2208_11469_b200/_lib
for v in l2h2 l2h1; do
PG_LIB_PATH=$PWD/$L/$v/libprobgraph_b200.so timeout 900 ncu -f --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_bloom -s 1 -c 1 python scripts/prof_once.py c5 2>&1 | grep -E "dram__|gpu__time|hit_rate" | sed "s/^/$v /"
done
timeout 900 ncu -f --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_bloom -s 1 -c 1 python scripts/prof_once.py c5 2>&1 | grep -E "dram__|gpu__time|hit_rate" | sed "s/^/default /"
