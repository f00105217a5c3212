#!/usr/bin/env bash
# final build: sanitizers over every production kernel + the ncu launch list at 1e17
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
bash tools/gpu/sanitize.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02h_launches_e17.csv python tools/prof_job.py 1e17 1 > gpurun_out/r02h_launches_e17.log 2>&1
echo "launch list rc=$?"; tail -1 gpurun_out/r02h_launches_e17.log | grep -o "'kernel_launches': [0-9]*"
python tools/ncu_summary.py launches gpurun_out/r02h_launches_e17.csv | head -14
