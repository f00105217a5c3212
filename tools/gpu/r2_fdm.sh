#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for v in fdm64 fdm128; do MT_LIB=tools/ab/lib_$v.so timeout 600 python -m pytest tests -m gpu -x -q -k "production or wheel or small_n or paper_1e19" 2>&1 | tail -1; done
for L in paper_1108_0135_b200/libmertens_sm100.so tools/ab/lib_fdm64.so tools/ab/lib_fdm128.so; do
  MT_LIB=$L timeout 600 python tools/sieve_bench.py 2.3e12 20 4.64e12 2>&1 | grep "wheel 6"
  MT_LIB=$L timeout 600 python tools/sieve_bench.py 3e14 20 4.64e14 2>&1 | grep "wheel 6"
done
bash tools/ab/time_variants.sh 1e19 2 2>&1
