#!/usr/bin/env bash
# counted / dense split sweep: xcut = max(D, alpha * ceil(sqrt v)) vs the reference's split;
# correctness (M(1e19) and parity tests at one alpha) and per-kernel device time
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
MT_XCUT_ALPHA=0.3 timeout 900 python -m pytest tests -m gpu -x -q -k "small_n or seeded or paper_1e16 or paper_1e19 or multi or golden" 2>&1 | tail -1
for a in 0 0.2 0.25 0.3 0.35 0.4 0.5; do
  echo "== alpha $a"
  MT_XCUT_ALPHA=$a MT_TIMING=1 timeout 600 python tools/prof_job.py 1e19 2 2>&1 | tail -1 | python -c "
import sys, ast
line = sys.stdin.read()
head, d = line.split(' {', 1)
d = ast.literal_eval('{' + d)
print(head, {k: round(v, 1) for k, v in d['kernel_ms'].items() if v}, 'head', round(d['ms_update_head']), 'tail', round(d['ms_sieve_tail']), 'q', round(d['ms_qgather']), 'total', round(d['ms_total']), 'nhead', d['n_head_segments'])"
done
