#!/usr/bin/env bash
# fill write-combining A/B (MT_FILL_BIN=0 -> direct stores), then parity tests
cd "$(dirname "$0")/../.."
for b in 0 128 0 128; do
  echo "bin=$b"
  MT_FILL_BIN=$b timeout 120 python tools/sieve_bench.py 2.3e12 40 4.64e12
  MT_FILL_BIN=$b timeout 120 python tools/sieve_bench.py 1.0e14 20 2.15e14
  MT_FILL_BIN=$b timeout 120 python tools/sieve_bench.py 3.0e14 10 4.64e14
done
for b in 0 128; do echo "== bin $b"; MT_FILL_BIN=$b MT_TIMING=1 timeout 200 python tools/prof_job.py 1e18 1 | grep -o "'kernel_ms.*" | cut -c1-300; done
timeout 900 python -m pytest tests -m gpu -x -q -k "sieve or prefix or golden or quotient or shard or e16 or checkpoint" 2>&1 | tail -3
