#!/bin/bash
# ncu evidence for the N=1 bench (B200_PROFILING.md recipe).  Runs on a GPU box:
#   1. the plain command (must exit 0 before any ncu run),
#   2. the launch list (gpu__time_duration per launch of our kernels),
#   3. one --set full capture of the top kernel (3 launches after warm-up).
# Usage: tools/ncu_profile.sh <tag> <kernel-regex> <skip> <count> [extra bench args...]
set -u
TAG=$1; KRE=$2; SKIP=$3; CNT=$4; shift 4
CMD="python bench.py --steps 1 --warmup 3 --no-corun --no-e2e --no-cpu-baseline $*"
mkdir -p gpurun_out
$CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/ncu_plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'pack|xor|signal' -c 1000 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c $CNT \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
ls -la gpurun_out/ | grep -E "$TAG"
