# The round-end measurement set (run on the GPU box via gpurun): the full bench line,
# the ncu launch list of the bench step, and an ncu --set full capture of the config-2 op
# kernels. Summarise with scripts/summarize_launches.py / scripts/summarize_ncu.py into profiles/.
python bench.py > gpurun_out/round_bench.json 2> gpurun_out/round_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 450 --csv --log-file gpurun_out/round_launches.csv python bench.py --steps 2 --warmup 1 --no-ops --no-cpu --no-bf16 > gpurun_out/round_launches.log 2>&1
ncu --set full --clock-control none -o gpurun_out/round_ops python scripts/prof_ops.py > gpurun_out/round_ops.log 2>&1
