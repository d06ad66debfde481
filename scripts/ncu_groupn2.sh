# DRAM bytes and time of the config-5 forward GEMM per raster group width (dynamic draws)
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct"
for gn in 8 16 2; do
  B2_GEMM_GROUPN=$gn ncu --clock-control none --metrics $M -k regex:k_gemm_tc --launch-skip 1 -c 1 --csv python scripts/epi_case.py fwd_split_only > gpurun_out/ncu_gn${gn}.csv 2>&1
done
for r in 1 2; do
  for gn in 8 16; do
    B2_GEMM_GROUPN=$gn timeout 200 python scripts/step_gemms.py --batch 65536 --steps 10 2>/dev/null | head -1 | sed "s/^/gn=$gn: /"
  done
done
