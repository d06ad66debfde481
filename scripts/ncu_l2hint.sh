# DRAM bytes and time of the config-5 forward GEMM under the L2 hint variants
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct"
for h in 1 2; do
  for gn in 8 4; do
    B2_GEMM_GROUPN=$gn B2_GEMM_L2HINT=$h ncu --clock-control none --metrics $M -k regex:k_gemm_tc --launch-skip 1 -c 1 --csv python scripts/epi_case.py fwd_split_only > gpurun_out/ncu_h${h}_gn${gn}.csv 2>&1
  done
done
