#!/usr/bin/env bash
# quick: M(1e16), M(1e19) with per-kernel times (and any tools/ab variants), + the golden e10 test
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "e10_full or multi_vs_oracle or forced_wide" 2>&1 | tail -2
bash tools/ab/time_variants.sh ${1:-1e19} ${2:-1}
