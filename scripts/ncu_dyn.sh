# DRAM bytes / time of the config-5 forward GEMM: static raster vs dynamic unit draws, raster widths
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct"
for gn in 8 16 4; do
for d in 0 1; do
  B2_GEMM_GROUPN=$gn B2_GEMM_DYNAMIC=$d ncu --clock-control none --metrics $M -k regex:k_gemm_tc --launch-skip 1 -c 1 --csv python scripts/epi_case.py fwd_split_only > gpurun_out/ncu_dyn${d}_gn$gn.csv 2>&1
done; done
