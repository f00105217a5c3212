#!/usr/bin/env bash
# bucket threshold sweep (primes above 2^b go to the bucket lists)
cd "$(dirname "$0")/../.."
for b in 15 16 17; do
  echo "== big 2^$b"
  MT_S2_BIG_LOG2=$b timeout 300 python tools/sieve_bench.py 2.3e12 20 4.64e12 2>&1 | grep "wheel 6"
  MT_S2_BIG_LOG2=$b timeout 300 python tools/sieve_bench.py 3e14 20 4.64e14 2>&1 | grep "wheel 6"
  MT_S2_BIG_LOG2=$b MT_TIMING=1 timeout 600 python tools/prof_job.py 1e19 2 2>&1 | tail -1 | cut -c1-260
done
MT_S2_BIG_LOG2=17 timeout 600 python -m pytest tests -m gpu -x -q -k "production or wheel or paper_1e19" 2>&1 | tail -1
