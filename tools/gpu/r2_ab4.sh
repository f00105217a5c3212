#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sieve or wheel or small_n or seeded or paper_1e16 or paper_1e19 or segment_size or multi or forced_wide or production or e10_full or ac2 or u_invariance" 2>&1 | tail -3
bash tools/ab/time_variants.sh 1e19 1 2>&1 | tee gpurun_out/ab4.txt
