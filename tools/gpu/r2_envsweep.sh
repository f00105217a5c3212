#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
for env in "X=1" "MT_SEG_TILES_PER_SM_HEAD=1" "MT_SEG_TILES_PER_SM_HEAD=4" "MT_SEG_TILES_PER_SM=8" "MT_QBLOCK_LOG2=23" "MT_QBLOCK_LOG2=25"; do
  echo "== $env"
  env $env MT_TIMING=1 timeout 600 python tools/prof_job.py 1e19 2 2>&1 | tail -1 | python -c "
import sys, ast
line = sys.stdin.read()
head, d = line.split(' {', 1)
d = ast.literal_eval('{' + d)
print(head, {k: round(v, 1) for k, v in d['kernel_ms'].items() if v}, 'head', round(d['ms_update_head']), 'tail', round(d['ms_sieve_tail']), 'q', round(d['ms_qgather']))"
done
