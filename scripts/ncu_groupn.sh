M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum"
for gn in 4 8 16; do
 for h in 1 0; do
  B2_GEMM_GROUPN=$gn B2_GEMM_L2HINT=$h ncu --clock-control none --metrics $M -k regex:k_gemm_tc --launch-skip 1 -c 1 --csv python scripts/epi_case.py fwd_split_only > gpurun_out/ncu_gn${gn}_h${h}.csv 2>&1
 done
done
