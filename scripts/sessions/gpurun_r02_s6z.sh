set -x
L=paper_2208_11469_b200/_lib
run() { echo "$1" >> gpurun_out/s6z_kern.log; shift; env "$@" timeout 600 python scripts/time_kernels.py c3kmv 2>&1 | tail -1 >> gpurun_out/s6z_kern.log; }
run "default" X=1
run "variant1 (16 warps, 128 regs)" PG_TMERGE_VARIANT=1
run "nu16" PG_LIB_PATH=$PWD/$L/nu16/libprobgraph_b200.so
run "nu16 variant1" PG_LIB_PATH=$PWD/$L/nu16/libprobgraph_b200.so PG_TMERGE_VARIANT=1
run "chunk512" PG_LIB_PATH=$PWD/$L/ch512/libprobgraph_b200.so
run "carve 80" PG_TMERGE_CARVEOUT=80
cat gpurun_out/s6z_kern.log
