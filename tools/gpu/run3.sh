cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r3_pytest.txt
cat gpurun_out/r3_pytest.txt
for e in 1e16 1e17 1e18 1e19; do timeout 300 python tools/prof_job.py $e 1 ; done > gpurun_out/r3_scale.txt 2>&1
cat gpurun_out/r3_scale.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sieve2 -s 200 -c 1 -o gpurun_out/r3_sieve2 python tools/prof_job.py 1e17 1 > gpurun_out/r3_ncu1.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bucket_fill -s 200 -c 1 -o gpurun_out/r3_bucket python tools/prof_job.py 1e17 1 > gpurun_out/r3_ncu2.txt 2>&1
tail -2 gpurun_out/r3_ncu1.txt gpurun_out/r3_ncu2.txt
