#!/usr/bin/env bash
# round-end style check on the final build, then ncu evidence of every top kernel
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
bash tools/gpu/r2_final.sh
bash tools/gpu/r2_ncu.sh r02e 2>&1 | tail -5
