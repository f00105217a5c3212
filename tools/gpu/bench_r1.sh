cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
cat gpurun_out/bench_r1.json; tail -3 gpurun_out/bench_r1.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_r1_ref.json 2>&1; cat gpurun_out/bench_r1_ref.json | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_e17.csv python tools/prof_job.py 1e17 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sieve3 -s 2000 -c 1 -o gpurun_out/r1_top_sieve3 python tools/prof_job.py 1e19 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_counted$' -s 60 -c 1 -o gpurun_out/r1_counted python tools/prof_job.py 1e19 1 > /dev/null 2>&1
echo done
