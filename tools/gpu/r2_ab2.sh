#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
df -h /dev/shm /tmp | tail -2; free -g | head -2; nproc
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "e10_full or multi_vs_oracle or forced_wide or segment_size" 2>&1 | tail -2
bash tools/ab/time_variants.sh 1e19 1
timeout 900 python tools/qmap_run.py 1e18 /dev/shm/qmap_e18; echo "qmap shm rc=$?"
