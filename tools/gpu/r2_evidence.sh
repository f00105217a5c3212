#!/usr/bin/env bash
# round-2 evidence: ncu (launch list + top kernels) and compute-sanitizer
cd "$(dirname "$0")/../.."
bash tools/gpu/r2_ncu.sh ${1:-r02b}
bash tools/gpu/sanitize.sh
