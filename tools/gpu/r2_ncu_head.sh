#!/usr/bin/env bash
# ncu --set full of the first head segment's update kernels (where 90 % of their work is)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
T=${1:-r02c}
for k in k_counted:0 k_dwin:0 k_dsparse:1; do
  name=${k%%:*}; skip=${k##*:}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^${name}$" -s $skip -c 1 \
    -o gpurun_out/${T}_${name} -f python tools/prof_job.py 1e19 1 > gpurun_out/${T}_${name}.log 2>&1
  echo "$name rc=$?"
done
python tools/ncu_summary.py rep gpurun_out/${T}_k_*.ncu-rep
