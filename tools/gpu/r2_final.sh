#!/usr/bin/env bash
# round-end style check: smoke, the whole GPU suite (incl. slow), the bench line, the
# 2-rank gloo bench on one GPU, the reference arm
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
export MT_RESULTS_DIR=$PWD/gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 3600 python -m pytest tests -q -m gpu --durations=20 > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"
tail -28 gpurun_out/final_pytest.log
timeout 1500 python bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 1500 python bench.py --gpus 2 --dist-backend gloo --steps 2 --warmup 3 --no-anchor > gpurun_out/final_bench2g.json 2> gpurun_out/final_bench2g.err; echo "bench2 rc=$?"
timeout 1500 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/final_bench.json", "gpurun_out/final_bench2g.json", "gpurun_out/final_bench_ref.json"):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    except Exception as ex:
        print(f, "failed", ex); continue
    print(f, {k: d.get(k) for k in ("value", "ms_per_step", "n_gpus", "gpu_launches")}, d.get("result"),
          (d.get("e2e") or {}).get("value"), (d.get("anchor") or {}).get("value"), d.get("kernel_ms_per_step"))
PY
