#!/bin/bash
# ncu --set full captures of the stage kernels (one step) with per-line source pages.
#   bash scripts/ncu_r02.sh <tag> <config> <arith> <count>
TAG=$1; CFG=$2; AR=${3:-fast}; C=${4:-4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -c $C \
   -o $OUT/prof_${CFG//:/_} python scripts/ncu_target.py $CFG $AR 1 > $OUT/ncu_${CFG//:/_}.log 2>&1
python scripts/ncu_summary.py $OUT/prof_${CFG//:/_}.ncu-rep $OUT/ncu_${CFG//:/_}.json > /dev/null 2>&1
for k in ${KS:-$(seq 1 $C)}; do
  ncu -i $OUT/prof_${CFG//:/_}.ncu-rep --page source --csv --print-source cuda,sass --launch-skip $((k-1)) --launch-count 1 \
     > $OUT/src_${CFG//:/_}_$k.csv 2>/dev/null
done
gzip -f $OUT/src_*.csv
find $OUT -name '*.ncu-rep' -size +${KEEPREP:-20}M -delete
ls -la $OUT
