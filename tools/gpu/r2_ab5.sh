#!/usr/bin/env bash
# paired-list sieve + vector counted walk: parity subset, bench line, ncu of the two kernels
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sieve or wheel or small_n or seeded or paper_1e16 or paper_1e19 or segment_size or multi or forced_wide or production or e10_full or ac2 or u_invariance or sharded or checkpoint or paper_1e20" 2>&1 | tail -3
timeout 1500 python bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err; echo "bench rc=$?"
tail -2 gpurun_out/bench_r02d.err
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/bench_r02d.json") if l.startswith("{")][-1])
print({k: d.get(k) for k in ("value", "ms_per_step", "gpu_launches")}, d.get("result"), d.get("e2e", {}).get("value"), d.get("kernel_ms_per_step"), d.get("clocks"))
PY
T=r02d
for k in k_sieve3:5000 k_counted:0; do
  name=${k%%:*}; skip=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${name}(<[0-9]+>)?$" -s $skip -c 1 \
    -o gpurun_out/${T}_${name} -f python tools/prof_job.py 1e19 1 > gpurun_out/${T}_${name}.log 2>&1
  echo "$name rc=$?"
done
python tools/ncu_summary.py rep gpurun_out/${T}_k_*.ncu-rep > gpurun_out/${T}_ncu_summary.txt; head -60 gpurun_out/${T}_ncu_summary.txt
