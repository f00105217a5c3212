#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
for big in 17 16; do
  echo "BIG_LOG2=$big"
  MT_S2_BIG_LOG2=$big timeout 120 python tools/sieve_bench.py 2.3e12 40 4.64e12
  MT_S2_BIG_LOG2=$big timeout 120 python tools/sieve_bench.py 3.0e14 10 4.64e14
done
for t in 4 2 8; do echo "== tiles/SM $t"; MT_SEG_TILES_PER_SM=$t MT_TIMING=1 timeout 200 python tools/prof_job.py 1e18 1 | grep -o "'kernel_ms.*" | cut -c1-260; done
