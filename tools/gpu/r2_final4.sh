#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
bash tools/gpu/r2_final.sh
timeout 3000 python tools/paper_run.py 1e22 > gpurun_out/r02_paper_e22_final.json 2> gpurun_out/r02_paper_e22_final.err; echo "paper rc=$?"
cat gpurun_out/r02_paper_e22_final.json | cut -c1-900
