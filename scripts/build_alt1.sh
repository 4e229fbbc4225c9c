#!/bin/bash
# A/B build of the engine with ONE source file recompiled under extra defines:
#   scripts/build_alt1.sh NAME pg_minhash "-DPG_OH_FILTER=0"  ->  _lib/NAME/libprobgraph_b200.so
set -e
cd "$(dirname "$0")/../paper_2208_11469_b200/csrc"
name=$1; src=$2; defs=$3
mkdir -p ../_lib/$name
nvcc -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Xptxas -v \
  -gencode arch=compute_100a,code=sm_100a -I../../include $defs -dc -c $src.cu -o ../_lib/$name/$src.o 2> ../_lib/$name/ptxas.log
objs=$(ls ../_lib/obj/*.o | grep -v /$src.o | grep -v /${src%_old}.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $objs ../_lib/$name/$src.o -o ../_lib/$name/libprobgraph_b200.so -lcudart_static -lrt -lpthread -ldl
