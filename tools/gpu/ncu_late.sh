#!/usr/bin/env bash
# ncu --set full of one late-tail k_bucket_fill and k_sieve3 launch of mertens_exact(1e19)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
T=${1:-rl}
for k in k_bucket_fill:55000 k_sieve3:55000; do
  name=${k%%:*}; skip=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${name}$" -s $skip -c 1 \
    -o gpurun_out/${T}_${name} -f python tools/prof_job.py 1e19 1 > gpurun_out/${T}_${name}.log 2>&1
done
ls -la gpurun_out/ | grep "${T}_"
