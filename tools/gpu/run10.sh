cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sieve3 -s 14000 -c 1 -o gpurun_out/r10_sieve3_e19 python tools/prof_job.py 1e19 1 > /dev/null 2>&1
echo done
