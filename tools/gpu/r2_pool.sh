#!/usr/bin/env bash
# pooled device allocations: parity + where the end-to-end time goes with and without the pool
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "device_memory_pool or paper_1e19 or small_n or checkpoint or sharded or multi or memmap" 2>&1 | tail -2
echo "== MT_POOL=0"; MT_POOL=0 timeout 600 python tools/e2e_breakdown.py 1e19
echo "== pool"; timeout 600 python tools/e2e_breakdown.py 1e19
