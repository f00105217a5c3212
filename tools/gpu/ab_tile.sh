#!/usr/bin/env bash
# tile-kernel A/B: in-tree library vs tools/variants/lib_*.so, then parity tests
cd "$(dirname "$0")/../.."
for i in 1 2; do
  for v in main $(ls tools/variants 2>/dev/null | sed 's/lib_\(.*\)\.so/\1/'); do
    if [ $v = main ]; then unset MT_LIB; else export MT_LIB=tools/variants/lib_$v.so; fi
    echo "[$v]"
    timeout 120 python tools/sieve_bench.py 2.3e12 40 4.64e12
    timeout 120 python tools/sieve_bench.py 3.0e14 10 4.64e14
  done
done
unset MT_LIB
timeout 900 python -m pytest tests -m gpu -x -q -k "sieve or prefix or golden or quotient or shard or e16 or checkpoint" 2>&1 | tail -2
