cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sieve2 -s 30000 -c 1 -o gpurun_out/r8_sieve2_e19 python tools/prof_job.py 1e19 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bucket_fill -s 30000 -c 1 -o gpurun_out/r8_bucket_e19 python tools/prof_job.py 1e19 1 > /dev/null 2>&1
echo done
