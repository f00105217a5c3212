#!/usr/bin/env bash
# Build engine variants with extra -D flags into tools/variants/lib_<name>.so
# usage: tools/variants.sh name "-DFOO=1" [name2 "-DBAR=0" ...]
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
mkdir -p "$ROOT/tools/variants"
C="$ROOT/paper_1108_0135_b200/csrc"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $flags \
    -o "$ROOT/tools/variants/lib_$name.so" "$C/mt_engine.cu" "$C/mt_sieve.cu" "$C/mt_sieve2.cu" "$C/mt_update.cu" &
done
wait
ls -la "$ROOT/tools/variants"
