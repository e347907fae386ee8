# ring-depth sweep (tuning): per-stage ms, arith given as $1 (0 exact, 1 fast)
for D in auto 0 2; do
  if [ $D = auto ]; then unset NDGX_DEPTH; else export NDGX_DEPTH=$D; fi
  timeout 200 python scripts/quickbench.py ${1:-1} 2>&1 | grep 'rk' | cut -c1-210 | sed "s/^/depth=$D /"
done
