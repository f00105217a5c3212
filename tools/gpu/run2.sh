set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r2_pytest.txt
timeout 300 python tools/prof_job.py 1e19 1 > gpurun_out/r2_e19.txt 2>&1
timeout 600 python bench.py --n 1e17 --warmup 3 --steps 2 > gpurun_out/r2_bench_e17.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_e16.csv python tools/prof_job.py 1e16 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sieve_tile -s 60 -c 1 -o gpurun_out/r2_sieve_tile python tools/prof_job.py 1e17 1 > gpurun_out/r2_ncu1.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sieve_large -s 60 -c 1 -o gpurun_out/r2_sieve_large python tools/prof_job.py 1e17 1 > gpurun_out/r2_ncu2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_counted -s 8 -c 1 -o gpurun_out/r2_counted python tools/prof_job.py 1e17 1 > gpurun_out/r2_ncu3.txt 2>&1
cat gpurun_out/r2_pytest.txt gpurun_out/r2_e19.txt gpurun_out/r2_bench_e17.txt; tail -3 gpurun_out/r2_ncu*.txt
