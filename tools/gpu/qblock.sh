#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -2
for b in 40 24 23 25 22; do
  echo "qblock 2^$b"; MT_QBLOCK_LOG2=$b MT_TIMING=1 timeout 300 python tools/prof_job.py 1e19 1 | grep -o "^10000000000000000000 [-0-9]*\|'qgather': [0-9.]*\|'ms_qgather': [0-9.]*"
done
