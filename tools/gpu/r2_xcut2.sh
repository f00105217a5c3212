#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
MT_XCUT_ALPHA=0.42 timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -1
for r in 1 2; do
for a in 0 0.38 0.4 0.42 0.45; do
  echo "== alpha $a"
  MT_XCUT_ALPHA=$a MT_TIMING=1 timeout 600 python tools/prof_job.py 1e19 2 2>&1 | tail -1 | python -c "
import sys, ast
line = sys.stdin.read()
head, d = line.split(' {', 1)
d = ast.literal_eval('{' + d)
print(head, {k: round(v, 1) for k, v in d['kernel_ms'].items() if v}, 'head', round(d['ms_update_head']), 'tail', round(d['ms_sieve_tail']), 'q', round(d['ms_qgather']), 'total', round(d['ms_total']), 'nhead', d['n_head_segments'])"
done
done
MT_XCUT_ALPHA=0.42 MT_TIMING=1 timeout 900 python tools/prof_job.py 1e20 1 2>&1 | tail -1 | cut -c1-300
MT_TIMING=1 timeout 900 python tools/prof_job.py 1e20 1 2>&1 | tail -1 | cut -c1-300
