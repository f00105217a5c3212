cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sieve2 -s 30000 -c 1 -o gpurun_out/r5_sieve2_e19 python tools/prof_job.py 1e19 1 > gpurun_out/r5_a.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bucket_fill -s 30000 -c 1 -o gpurun_out/r5_bucket_e19 python tools/prof_job.py 1e19 1 > gpurun_out/r5_b.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_(counted|dwin|dsparse)$' -s 180 -c 3 -o gpurun_out/r5_update_e19 python tools/prof_job.py 1e19 1 > gpurun_out/r5_c.txt 2>&1
tail -n 3 gpurun_out/r5_a.txt gpurun_out/r5_b.txt gpurun_out/r5_c.txt
