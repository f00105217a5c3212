#!/usr/bin/env bash
# ncu evidence: launch list of one mertens_exact(1e17) (kernel shares + launch count)
# and one --set full capture of each top kernel inside mertens_exact(1e19)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
T=${1:-r02}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches_e17.csv python tools/prof_job.py 1e17 1 > gpurun_out/${T}_launches_e17.log 2>&1
echo "launch list rc=$?"; tail -2 gpurun_out/${T}_launches_e17.log | cut -c1-400
python tools/ncu_summary.py launches gpurun_out/${T}_launches_e17.csv | head -20
# skips: 1e19 has 221 head segments and ~13300 odd tail segments (3 sieve launches each)
for k in k_sieve3:5000 k_bucket_fill:5000 k_s3_finish:5000 k_counted:60 k_dwin:60 k_dsparse:60 k_qitems:2; do
  name=${k%%:*}; skip=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${name}(<[0-9]+>)?$" -s $skip -c 1 \
    -o gpurun_out/${T}_${name} -f python tools/prof_job.py 1e19 1 > gpurun_out/${T}_${name}.log 2>&1
  echo "$name rc=$?"
done
python tools/ncu_summary.py json gpurun_out/${T}_ncu_metrics.json gpurun_out/${T}_k_*.ncu-rep > /dev/null
python tools/ncu_summary.py rep gpurun_out/${T}_k_*.ncu-rep > gpurun_out/${T}_ncu_summary.txt
cat gpurun_out/${T}_ncu_summary.txt | head -120
