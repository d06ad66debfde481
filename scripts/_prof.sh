python bench.py > gpurun_out/bench_r01k.json 2> gpurun_out/bench_r01k.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 450 --csv --log-file gpurun_out/r01k_launches.csv python bench.py --steps 2 --warmup 1 --no-ops --no-cpu --no-bf16 > gpurun_out/r01k_launches.log 2>&1
ncu --set full --clock-control none -o gpurun_out/r01k_ops python scripts/prof_ops.py > gpurun_out/r01k_ops.log 2>&1
