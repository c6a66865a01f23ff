#!/bin/bash
# Usage (on the GPU box via gpurun): bash profiles/ncu_capture.sh <tag> [bench args...]
# 1) plain run (must exit 0), 2) launch list (gpu__time_duration per launch),
# 3) one --set full capture of the back-projection kernel.
set -u
TAG=$1; shift
ARGS="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary $*"
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain_$TAG.log; exit 1; }
tail -1 gpurun_out/plain_$TAG.log
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
    -k 'regex:cbb::|FillFunctor' --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list exit=$?"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:cbb::bp_(tma_)?kernel' -s 20 -c 1 -o gpurun_out/prof_$TAG -f \
    python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full capture exit=$?"
