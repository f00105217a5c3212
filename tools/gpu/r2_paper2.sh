#!/usr/bin/env bash
# paper-scale evidence on the final build: M(1e20), M(1e21), M(1e22) with quotients
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 4000 python tools/paper_run.py 1e20 1e21 1e22 > gpurun_out/r02_paper_final.json 2> gpurun_out/r02_paper_final.err; echo "paper rc=$?"
cat gpurun_out/r02_paper_final.json; tail -3 gpurun_out/r02_paper_final.err
