#!/bin/bash
# Build an A/B variant of libtetris_b200.so with extra nvcc flags into paper_2502_15197_b200/_native/<name>
# usage: bash tools/build_variant.sh NAME "-DFLAG ..."   then run with TETRIS_LIB_VARIANT=NAME
set -e
NAME=$1; FLAGS=$2
R=$(cd "$(dirname "$0")/.." && pwd)
OUT=$R/paper_2502_15197_b200/_native/var_$NAME
mkdir -p $OUT
for f in abi select select1 gselect verify stream greedy compact sim dist; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -I $R/include $FLAGS -c $R/paper_2502_15197_b200/csrc/$f.cu -o $OUT/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $R/paper_2502_15197_b200/_native/$NAME $OUT/*.o -ldl
echo built $R/paper_2502_15197_b200/_native/$NAME
