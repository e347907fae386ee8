#!/bin/bash
# GPU-scale sweeps through the reference-schema drivers.
# Reports land in gpurun_out/exp/ (copy the ones worth keeping to profiles/).
OUT=gpurun_out/exp; mkdir -p $OUT
E="python -m paper_2510_05254_b200.experiments"
# convergence of 2D advection at order 4/6/8 up to 256^2 cells (t_end = 1)
timeout 600 $E converge --dim 2 --order 4 --order 6 --order 8 --rk rk6 --cells 8 --cells 16 --cells 32 \
  --cells 64 --cells 128 --cells 256 --nk 4 --seed 42 --out $OUT/converge_2d.csv
# fixed-step cost per DOF across orders, 2D Euler (+ advection), ~1e8 DOF, both arithmetic modes
for AR in exact fast; do
  timeout 600 $E timing --equation euler --dim 2 --order 3 --order 4 --order 6 --order 8 --rk rk4 \
    --cells 1536 --steps 20 --compare-equations --arith $AR --out $OUT/timing_2d_$AR.csv
  timeout 600 $E timing --equation euler --dim 3 --order 3 --order 4 --rk rk4 --cells 96 --steps 10 \
    --arith $AR --out $OUT/timing_3d_$AR.csv
done
ls -la $OUT
