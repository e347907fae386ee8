mkdir -p gpurun_out/bench1
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench1/bench.json 2> gpurun_out/bench1/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench1/bench_ref.json 2> gpurun_out/bench1/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench1/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-exact-arm > gpurun_out/bench1/ncu_bench.log 2>&1
cat gpurun_out/bench1/bench.json gpurun_out/bench1/bench_ref.json
