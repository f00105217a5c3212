#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "split_invariance or checkpoint or u_invariance" 2>&1 | tail -2
timeout 4000 python tools/paper_run.py 1e20 1e21 1e22 > gpurun_out/r02_paper_final2.json 2> gpurun_out/r02_paper_final2.err; echo "paper rc=$?"
cat gpurun_out/r02_paper_final2.json; tail -3 gpurun_out/r02_paper_final2.err
