#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "small_n or seeded or paper_1e16 or paper_1e19 or paper_1e20 or forced_wide or multi or split_invariance or sharded or checkpoint" 2>&1 | tail -1
for r in 1 2; do bash tools/ab/time_variants.sh 1e19 2 2>&1; done
