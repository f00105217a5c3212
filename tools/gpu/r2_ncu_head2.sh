#!/usr/bin/env bash
# ncu --set full of the first head segment's k_counted / k_dwin (the bulk of their work) on
# the final build, plus the fill padding change: parity subset and a timing pair
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "production or wheel or small_n or paper_1e19" 2>&1 | tail -1
bash tools/ab/time_variants.sh 1e19 2 2>&1 | tee gpurun_out/ab11.txt
T=r02f
for k in k_counted:0 k_dwin:0; do
  name=${k%%:*}; skip=${k##*:}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^${name}$" -s $skip -c 1 \
    -o gpurun_out/${T}_${name} -f python tools/prof_job.py 1e19 1 > gpurun_out/${T}_${name}.log 2>&1
  echo "$name rc=$?"
done
python tools/ncu_summary.py rep gpurun_out/${T}_k_*.ncu-rep > gpurun_out/${T}_ncu_head.txt; head -50 gpurun_out/${T}_ncu_head.txt
