python bench.py > gpurun_out/bench_r01j.json 2> gpurun_out/bench_r01j.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01j_launches.csv python bench.py --steps 2 --warmup 1 --no-ops --no-cpu --no-bf16 > gpurun_out/r01j_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc --launch-skip 1 -c 1 -o gpurun_out/r01j_gemm python scripts/epi_case.py fwd_split_only > gpurun_out/r01j_gemm.log 2>&1
ncu --set full --clock-control none -o gpurun_out/r01j_ops python scripts/prof_ops.py > gpurun_out/r01j_ops.log 2>&1
