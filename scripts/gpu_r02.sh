#!/bin/bash
# Round-2 GPU baseline: smoke, GPU tests, bench lines for every config, reference arm, launch list.
#   bash scripts/gpu_r02.sh <tag> [skip-tests]
TAG=${1:-r02}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/smi.txt 2>&1
lscpu | head -20 > $OUT/lscpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
if [ "$2" != "skip-tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q --timeout 200 > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
  tail -6 $OUT/pytest.log
fi
for c in c3 c2 c4 c5; do
  case $c in c4) K=6;; c5) K=10;; *) K=30;; esac
  timeout 600 python bench.py --config $c --steps $K --warmup 3 $([ $c != c3 ] && echo --no-cpu-baseline --no-exact-arm) \
     > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "$c: $(head -c 600 $OUT/bench_$c.json)"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-exact-arm > $OUT/ncu_bench.log 2>&1
echo done
