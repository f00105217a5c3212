#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -2
MT_TIMING=1 timeout 300 python tools/prof_job.py 1e19 1 | grep -o "^10000000000000000000 [-0-9]* [0-9.]*s\|'kernel_ms.*" | cut -c1-300
