#!/usr/bin/env bash
# window/sparse split cap C in d_sp = ceil(sqrt(v)/min(C, cbrt(sqrt(v)/2)))
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for v in ws32 ws128 ws256; do MT_LIB=tools/ab/lib_$v.so timeout 600 python -m pytest tests -m gpu -x -q -k "small_n or seeded or paper_1e19 or forced_wide" 2>&1 | tail -1; done
for r in 1 2; do bash tools/ab/time_variants.sh 1e19 2 2>&1; done | tee gpurun_out/ab_ws.txt
