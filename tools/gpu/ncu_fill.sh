#!/usr/bin/env bash
# ncu --set full of one k_bucket_fill and one k_sieve3 launch of a tail segment
# usage: ncu_fill.sh TAG [Y0=2.3e12] [YLAST=4.64e12] [what=fill,s3]
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
tag=${1:-fill}; Y0=${2:-2.3e12}; YL=${3:-4.64e12}; what=${4:-fill,s3}
if [[ $what == *fill* ]]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bucket_fill -s 10 -c 1 \
  -o gpurun_out/${tag}_fill -f python tools/sieve_bench.py $Y0 8 $YL >> gpurun_out/${tag}_ncu.log 2>&1
fi
if [[ $what == *s3* ]]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sieve3 -s 10 -c 1 \
  -o gpurun_out/${tag}_s3 -f python tools/sieve_bench.py $Y0 8 $YL >> gpurun_out/${tag}_ncu.log 2>&1
fi
ls -la gpurun_out/${tag}_*
