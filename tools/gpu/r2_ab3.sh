#!/usr/bin/env bash
# sieve/fill rewrite: parity subset, A/B of the variants, the 1e19 quotient-map residual
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sieve or wheel or small_n or seeded or paper_1e16 or paper_1e19 or segment_size or multi or sharded or production or e10_full" 2>&1 | tail -3
bash tools/ab/time_variants.sh 1e19 1 2>&1 | tee gpurun_out/ab3.txt
timeout 900 python tools/qmap_run.py 1e19 /dev/shm/qmap_e19 > gpurun_out/qmap_e19.json 2> gpurun_out/qmap_e19.err
echo "qmap rc=$?"; tail -3 gpurun_out/qmap_e19.err; cat gpurun_out/qmap_e19.json
