#!/usr/bin/env bash
# ncu --set full of k_bucket_fill / k_sieve3 on the final build (same launches as r02e)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
T=r02g
for k in k_bucket_fill:5000 k_sieve3:5000; do
  name=${k%%:*}; skip=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${name}(<[0-9]+>)?$" -s $skip -c 1 \
    -o gpurun_out/${T}_${name} -f python tools/prof_job.py 1e19 1 > gpurun_out/${T}_${name}.log 2>&1
  echo "$name rc=$?"
done
python tools/ncu_summary.py json gpurun_out/${T}_ncu_metrics.json gpurun_out/${T}_k_*.ncu-rep > /dev/null
python tools/ncu_summary.py rep gpurun_out/${T}_k_*.ncu-rep > gpurun_out/${T}_ncu_summary.txt; head -44 gpurun_out/${T}_ncu_summary.txt
