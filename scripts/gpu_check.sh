#!/bin/bash
# One GPU round-trip: parity tests, quick throughput table, one ncu capture.
#   bash scripts/gpu_check.sh <tag> [ncu-config] [ncu-arith]
TAG=${1:-dev}; CFG=${2:-c3}; AR=${3:-exact}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python scripts/quickbench.py 2>&1 | tail -12
if [ "$CFG" != "none" ]; then
  case $CFG in c4) S=7;; *) S=4;; esac
  timeout 500 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s $S -c $S \
     -o gpurun_out/prof_${CFG}_${AR}_${TAG} python scripts/ncu_target.py $CFG $AR 2 2>&1 | tail -1
fi
