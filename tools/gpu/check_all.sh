#!/usr/bin/env bash
# full non-slow GPU suite + a short bench line
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/chk_bench.json 2> gpurun_out/chk_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/chk_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'ms', d['ms_per_step'], d['result'], d['kernel_ms_per_step'], d['phases_ms'], d['roofline']['frac'])"
tail -3 gpurun_out/chk_bench.err
