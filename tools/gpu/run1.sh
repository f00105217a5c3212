set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r1_pytest.txt
for e in 1e13 1e14 1e15 1e16 1e17 1e18; do timeout 300 python tools/prof_job.py $e 2 ; done > gpurun_out/r1_scale.txt 2>&1
timeout 600 python tools/prof_job.py 1e19 1 >> gpurun_out/r1_scale.txt 2>&1
cat gpurun_out/r1_pytest.txt gpurun_out/r1_scale.txt
