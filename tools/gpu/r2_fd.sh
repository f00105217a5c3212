#!/usr/bin/env bash
# fill: short streams emitted in phase 1; parity + segment benchmarks at 1e19 and 1e22 ranges
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "production or wheel or small_n or seeded or paper_1e19 or paper_1e16" 2>&1 | tail -1
for L in paper_1108_0135_b200/libmertens_sm100.so tools/ab/lib_fd0.so; do
  MT_LIB=$L timeout 600 python tools/sieve_bench.py 2.3e12 20 4.64e12 2>&1 | grep "wheel 6"
  MT_LIB=$L timeout 600 python tools/sieve_bench.py 3e14 20 4.64e14 2>&1 | grep "wheel 6"
done
bash tools/ab/time_variants.sh 1e19 2 2>&1
