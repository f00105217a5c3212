#!/usr/bin/env bash
# the bench line (driver command) and the reference arm
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_r02.err
timeout 1500 python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/bench_r02_ref.json 2> gpurun_out/bench_r02_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/bench_r02.json", "gpurun_out/bench_r02_ref.json"):
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    print(f, {k: d.get(k) for k in ("value", "ms_per_step", "gpu_launches")}, d.get("result"), d.get("e2e", {}).get("value"),
          (d.get("anchor") or {}).get("value"), (d.get("anchor") or {}).get("wall_s"), d.get("kernel_ms_per_step"))
PY
