#!/bin/bash
# Tuning sweep: per-stage ms of every _variants/<name>/libndgx.so on the given configs.
#   bash scripts/var_bench.sh <out-tag> <configs> [pytest-filter]
TAG=${1:-var}; CF=${2:-c4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ -n "$3" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "$3" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log; tail -3 $OUT/pytest.log
fi
for v in $(ls _variants); do
  NDGX_LIB=_variants/$v/libndgx.so timeout 300 python scripts/stagebench.py $v $CF >> $OUT/stages.jsonl 2> $OUT/err_$v.log
done
timeout 300 python scripts/stagebench.py main $CF >> $OUT/stages.jsonl 2> $OUT/err_main.log
cat $OUT/stages.jsonl
