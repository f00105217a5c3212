#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
bash tools/ab/time_variants.sh 1e17 1
for lib in paper_1108_0135_b200/libmertens_sm100.so tools/ab/lib_old.so; do
  tag=$(basename $lib .so)
  MT_LIB=$lib timeout 900 ncu --section SchedulerStats --section WarpStateStats --section SourceCounters \
    --section ComputeWorkloadAnalysis --section LaunchStats --section InstructionStats --clock-control none \
    --import-source on -k regex:"^k_counted$" -s 0 -c 1 -o gpurun_out/probe_${tag} -f python tools/prof_job.py 1e17 1 > gpurun_out/probe_${tag}.log 2>&1
  echo "$tag rc=$?"
  ncu -i gpurun_out/probe_${tag}.ncu-rep --page details 2>/dev/null | grep -E "Duration|Issued Warp|Eligible Warps|Active Threads|Executed Instructions  |Warp Cycles Per Issued" | head -12
done
