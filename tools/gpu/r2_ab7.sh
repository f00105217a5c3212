#!/usr/bin/env bash
# wheel-6 counted walk: parity (everything that runs the counted kernel) + timing vs the odd-m build
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "small_n or seeded or paper_1e16 or paper_1e19 or paper_1e20 or multi or forced_wide or sharded or checkpoint or golden or reference_values or survey or u_invariance or segment_size or plan_phases or ac2 or naive or e10_full or tail_wheel" 2>&1 | tail -3
bash tools/ab/time_variants.sh 1e19 2 2>&1 | tee gpurun_out/ab7.txt
