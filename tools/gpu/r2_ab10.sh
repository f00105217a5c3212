#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "small_n or seeded or paper_1e19 or multi or sharded or checkpoint or production or wheel" 2>&1 | tail -2
for i in 1 2; do bash tools/ab/time_variants.sh 1e19 3 2>&1; done | tee gpurun_out/ab10.txt
