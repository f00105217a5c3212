#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
bash tools/gpu/r2_final.sh
bash tools/gpu/r2_ncu_head2.sh 2>&1 | tail -45
