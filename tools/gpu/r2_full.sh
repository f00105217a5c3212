#!/usr/bin/env bash
# full GPU suite (incl. slow), bench line (1 GPU), and the 2-rank gloo bench on the one GPU
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
export MT_RESULTS_DIR=$PWD/gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_all.log
timeout 1200 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
timeout 1200 python bench.py --gpus 2 --dist-backend gloo --steps 1 --warmup 3 --no-anchor > gpurun_out/bench2g.json 2> gpurun_out/bench2g.err; echo "bench2 rc=$?"
tail -c 1500 gpurun_out/bench2g.json; tail -5 gpurun_out/bench2g.err
