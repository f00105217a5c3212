#!/usr/bin/env bash
# build A/B variants of the engine library into tools/ab/lib_<name>.so
# usage: tools/ab/build_variants.sh name1 "-DFLAG=1 ..." name2 "..." ...
cd "$(dirname "$0")/../.."
S=paper_1108_0135_b200/csrc
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    $flags -o tools/ab/lib_${name}.so $S/mt_engine.cu $S/mt_sieve.cu $S/mt_sieve2.cu $S/mt_update.cu $S/mt_qsum.cu &
done
wait
ls -la tools/ab/*.so
