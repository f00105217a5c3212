#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
for i in 1 2; do
  timeout 120 python tools/sieve_bench.py 2.3e12 40 4.64e12
  timeout 120 python tools/sieve_bench.py 1.0e14 20 2.15e14
  timeout 120 python tools/sieve_bench.py 3.0e14 10 4.64e14
done
timeout 900 python -m pytest tests -m gpu -x -q -k "sieve or prefix or golden or quotient or shard or e16 or checkpoint" 2>&1 | tail -2
