#!/usr/bin/env bash
# time M(n) with per-kernel events for every tools/ab/lib_*.so (and the default build)
# usage: tools/ab/time_variants.sh [n=1e19] [reps=2]
cd "$(dirname "$0")/../.."
n=${1:-1e19}; reps=${2:-2}
for lib in paper_1108_0135_b200/libmertens_sm100.so $(ls tools/ab/lib_*.so 2>/dev/null); do
  echo "== $lib"
  MT_LIB=$lib MT_TIMING=1 timeout 900 python tools/prof_job.py $n $reps 2>&1 | tail -1 | python -c "
import sys, ast
line = sys.stdin.read()
head, d = line.split(' {', 1)
d = ast.literal_eval('{' + d)
print(head, {k: round(v, 1) for k, v in d['kernel_ms'].items() if v}, 'head', round(d['ms_update_head']), 'tail', round(d['ms_sieve_tail']))"
done
