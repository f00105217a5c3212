#!/usr/bin/env bash
# official bench line + reference arm + ncu evidence (launch list and top kernels)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
T=${1:-rf}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -1 gpurun_out/${T}_bench.json | cut -c1-400; tail -3 gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
tail -1 gpurun_out/${T}_bench_ref.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_e17.csv python tools/prof_job.py 1e17 1 > /dev/null 2>&1
for k in k_sieve3:2000 k_bucket_fill:2000 k_counted:5 k_dwin:5; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${name}$" -s $skip -c 1 \
    -o gpurun_out/${T}_${name} -f python tools/prof_job.py 1e19 1 > gpurun_out/${T}_${name}.log 2>&1
done
ls -la gpurun_out/ | grep "${T}_"
echo done
