#!/bin/bash
# One GPU round-trip: parity tests, throughput table, bench line, optional ncu.
#   bash scripts/gpu_round.sh <tag> [ncu: none|c3|c4] [arith]
TAG=${1:-dev}; NCU=${2:-none}; AR=${3:-exact}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/smi.txt 2>&1
timeout 90 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; RC=$?; echo "smoke rc=$RC" >> $OUT/smoke.log; tail -3 $OUT/smoke.log
if [ $RC -ne 0 ]; then echo "smoke failed: skipping the rest"; exit 1; fi
timeout 300 python -m pytest tests -m gpu -x -q --timeout 60 > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
timeout 400 python scripts/quickbench.py > $OUT/quick.log 2>&1; tail -8 $OUT/quick.log
if [ "$NCU" != "none" ]; then
  case $NCU in c4) S=7;; *) S=4;; esac
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s $S -c $S \
     -o $OUT/prof_${NCU}_${AR} python scripts/ncu_target.py $NCU $AR 2 > $OUT/ncu.log 2>&1
  python scripts/ncu_summary.py $OUT/prof_${NCU}_${AR}.ncu-rep $OUT/ncu_${NCU}_${AR}.json > /dev/null 2>&1
  ncu -i $OUT/prof_${NCU}_${AR}.ncu-rep --page source --csv > $OUT/src_${NCU}_${AR}.csv 2>/dev/null
  ls -la $OUT
  # keep the report only when small enough to travel back
  find $OUT -name '*.ncu-rep' -size +40M -delete
fi
