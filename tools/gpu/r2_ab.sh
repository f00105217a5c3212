#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
bash tools/ab/time_variants.sh 1e19 2
for t in 3 4 8; do
  echo "== MT_SEG_TILES_PER_SM=$t"
  MT_SEG_TILES_PER_SM=$t MT_TIMING=1 python tools/prof_job.py 1e19 2 2>&1 | tail -1 | cut -c1-60
done
