#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over every production kernel
# (tools/sanitize_job.py), logs into gpurun_out/ (summaries copied to profiles/)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
export MT_TEST_TILES=8
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  n=1e9; [ $tool = memcheck ] && n=1e11
  timeout 2400 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_job.py $n \
    > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_${tool}.log
done
