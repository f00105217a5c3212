#!/usr/bin/env bash
# paper-scale evidence: the dense quotient map of 1e19 (memory-mapped) with its identity
# residual, then M(1e20), M(1e21), M(1e22) with quotients
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
df -h /tmp | tail -1
timeout 1800 python tools/qmap_run.py 1e19 /tmp/qmap_e19 > gpurun_out/r02_qmap_e19.json 2> gpurun_out/r02_qmap_e19.err; echo "qmap rc=$?"
cat gpurun_out/r02_qmap_e19.json; tail -3 gpurun_out/r02_qmap_e19.err
timeout 4800 python tools/paper_run.py 1e20 1e21 1e22 > gpurun_out/r02_paper_e20_e22.json 2> gpurun_out/r02_paper.err; echo "paper rc=$?"
cat gpurun_out/r02_paper_e20_e22.json; tail -3 gpurun_out/r02_paper.err
