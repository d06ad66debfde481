# DRAM bytes and time of the config-5 forward GEMM with / without streaming
# (L2 evict-first) output stores, then the step alternated on the same box
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct"
for h in 1 5; do
  B2_GEMM_L2HINT=$h ncu --clock-control none --metrics $M -k regex:k_gemm_tc --launch-skip 1 -c 1 --csv python scripts/epi_case.py fwd_split_only > gpurun_out/ncu_stcs_h${h}.csv 2>&1
  B2_GEMM_L2HINT=$h ncu --clock-control none --metrics $M -k regex:k_gemm_tc --launch-skip 1 -c 1 --csv python scripts/epi_case.py full > gpurun_out/ncu_stcs_full_h${h}.csv 2>&1
done
for r in 1 2 3; do
  for h in 1 5; do
    B2_GEMM_L2HINT=$h timeout 200 python scripts/step_gemms.py --batch 65536 --steps 10 | head -1 | sed "s/^/h=$h: /"
  done
done
