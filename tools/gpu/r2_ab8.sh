#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "small_n or seeded or paper_1e19 or forced_wide" 2>&1 | tail -2
for v in cu8k; do MT_LIB=tools/ab/lib_$v.so timeout 600 python -m pytest tests -m gpu -x -q -k "small_n or seeded or paper_1e19 or forced_wide" 2>&1 | tail -1; done
bash tools/ab/time_variants.sh 1e19 2 2>&1 | tee gpurun_out/ab8.txt
