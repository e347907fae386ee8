# ring-depth sweep on the headline workload (tuning)
for D in auto 0 2 3 4; do
  if [ $D = auto ]; then unset NDGX_DEPTH; else export NDGX_DEPTH=$D; fi
  echo "depth=$D $(timeout 120 python scripts/quickbench.py 1 2>&1 | grep 'eq1 o8 rk1 arith1')"
done
