#!/bin/bash
# Round-2 final evidence: GPU tests, bench lines, reference arm, launch list, ncu summaries, overlap, sweep.
OUT=gpurun_out/${FINAL_TAG:-r02_final}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/smi.txt 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log; tail -3 $OUT/pytest.log
timeout 600 python bench.py --steps 30 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
for c in c2 c4 c5; do
  case $c in c4) K=8;; c5) K=10;; *) K=30;; esac
  timeout 600 python bench.py --config $c --steps $K --warmup 3 --no-cpu-baseline --no-exact-arm > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-exact-arm > $OUT/ncu_bench.log 2>&1
KS="1" bash scripts/ncu_r02.sh ${FINAL_TAG:-r02_final}/ncu_c3 c3 fast 4 > /dev/null 2>&1
KS="1" bash scripts/ncu_r02.sh ${FINAL_TAG:-r02_final}/ncu_c4 c4 fast 7 > /dev/null 2>&1
KS="1" bash scripts/ncu_r02.sh ${FINAL_TAG:-r02_final}/ncu_c2 c2 fast 4 > /dev/null 2>&1
find $OUT -name '*.ncu-rep' -delete
timeout 600 python scripts/overlap_bench.py > $OUT/overlap.jsonl 2>&1
timeout 600 python scripts/order_sweep.py final > $OUT/sweep.jsonl 2>&1
for c in c3 c2 c4 c5 ref; do echo "$c: $(head -c 300 $OUT/bench_$c.json)"; done
