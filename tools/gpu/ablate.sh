#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
for i in 1 2; do
for v in main $(ls tools/variants 2>/dev/null | sed 's/lib_\(.*\)\.so/\1/'); do
  if [ $v = main ]; then unset MT_LIB; else export MT_LIB=tools/variants/lib_$v.so; fi
  echo "[$v]"; timeout 120 python tools/sieve_bench.py 2.3e12 40 4.64e12
done
done
