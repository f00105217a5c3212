#!/usr/bin/env bash
# A/B of the bucket-list prefetch variants + the 1e19 dense quotient-map builder run
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
bash tools/ab/time_variants.sh 1e19 1 2>&1 | tee gpurun_out/ab_pf.txt
df -h /dev/shm | tail -1; free -g | head -2
timeout 1500 python tools/qmap_run.py 1e19 /dev/shm/qmap_e19 > gpurun_out/qmap_e19.json 2> gpurun_out/qmap_e19.err
echo "qmap rc=$?"; tail -3 gpurun_out/qmap_e19.err; cat gpurun_out/qmap_e19.json
