#!/usr/bin/env bash
# A/B of sieve variants (tools/variants/lib_*.so vs the in-tree library):
# sieve alone at the 1e19 tail and a 1e21-like tail, then whole 1e18 jobs.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for v in base vec main; do
  if [ $v = main ]; then unset MT_LIB; else export MT_LIB=tools/variants/lib_$v.so; fi
  timeout 120 python tools/sieve_bench.py 2.3e12 40 4.64e12
  timeout 120 python tools/sieve_bench.py 1.0e14 20 2.15e14
done
for v in base main base main; do
  if [ $v = main ]; then unset MT_LIB; else export MT_LIB=tools/variants/lib_$v.so; fi
  echo "== $v"; MT_TIMING=1 timeout 200 python tools/prof_job.py 1e18 1 | cut -c1-400
done
unset MT_LIB
timeout 900 python -m pytest tests -m gpu -x -q -k "sieve or prefix or golden or quotient or shard or e16" 2>&1 | tail -3
