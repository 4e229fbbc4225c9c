#!/bin/bash
# A/B build of the engine with pg_kmv.cu recompiled under extra defines:
#   scripts/build_kmv_alt.sh NAME "-DPG_TM_STEP2=1 ..."  ->  _lib/NAME/libprobgraph_b200.so
set -e
cd "$(dirname "$0")/../paper_2208_11469_b200/csrc"
name=$1; defs=$2
mkdir -p ../_lib/$name
nvcc -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Xptxas -v \
  -gencode arch=compute_100a,code=sm_100a -I../../include $defs -dc -c pg_kmv.cu -o ../_lib/$name/pg_kmv.o 2> ../_lib/$name/ptxas.log
objs=$(ls ../_lib/obj/*.o | grep -v pg_kmv.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $objs ../_lib/$name/pg_kmv.o -o ../_lib/$name/libprobgraph_b200.so -lcudart_static -lrt -lpthread -ldl
grep -A2 "tmerge_kernelILi64ELi8ELi20" ../_lib/$name/ptxas.log | grep -v Compiling | tr '\n' ' '; echo
