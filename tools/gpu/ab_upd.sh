#!/usr/bin/env bash
# update-kernel A/B: in-tree library vs tools/variants/lib_*.so at 1e19 (+ gpu tests for the in-tree one)
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -2
for v in main $(ls tools/variants 2>/dev/null | sed 's/lib_\(.*\)\.so/\1/'); do
  if [ $v = main ]; then unset MT_LIB; else export MT_LIB=tools/variants/lib_$v.so; fi
  echo "[$v]"; MT_TIMING=1 timeout 300 python tools/prof_job.py 1e19 1 | grep -o "^10000000000000000000 [-0-9]*\|'kernel_ms.*" | cut -c1-250
done
