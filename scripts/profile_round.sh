# The round's measurement set at HEAD (run on the GPU box via gpurun). Outputs go to
# gpurun_out/$TAG_*; summarise with scripts/summarize_launches.py / summarize_ncu.py into profiles/.
TAG=${TAG:-r02d}
O=gpurun_out
NCU="ncu --clock-control none"
# 1) the bench step's launch list (config 5, N=1)
$NCU --metrics gpu__time_duration.sum -c 450 --csv --log-file $O/${TAG}_step_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-ops --no-cpu --no-bf16 > $O/${TAG}_step_launches.log 2>&1
# 2) the dominant kernel, --set full: the config-5 hidden-layer forward GEMM as the step runs it
$NCU --set full --import-source on -k regex:k_gemm_tc --launch-skip 1 -c 1 -o $O/${TAG}_gemm_fwd -f \
  python scripts/epi_case.py fwd_split_only > $O/${TAG}_gemm_fwd.log 2>&1
# 3) config 3 (n = 1024, 4096) and config 4 launch lists with DRAM bytes
for n in 1024 4096; do
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
    --log-file $O/${TAG}_c3_n${n}_launches.csv python scripts/prof_c3.py $n > $O/${TAG}_c3_n${n}.log 2>&1
done
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $O/${TAG}_c4_launches.csv python scripts/prof_c4.py > $O/${TAG}_c4.log 2>&1
# 4) config-2 ops: per kernel (--set full) and the whole op set as one CUDA graph
$NCU --set full -o $O/${TAG}_ops -f python scripts/prof_ops.py > $O/${TAG}_ops.log 2>&1
$NCU --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --csv --log-file $O/${TAG}_ops_graph.csv python scripts/prof_ops_graph.py > $O/${TAG}_ops_graph.log 2>&1
# 5) the FP32 SIMT GEMM (FFMA2), --set full, n = 4096 in the forward layout; config-1 launch list
$NCU --set full --import-source on -k regex:k_gemm_simt --launch-skip 2 -c 1 -o $O/${TAG}_simt -f \
  python scripts/simt_one.py 4096 0 1 > $O/${TAG}_simt.log 2>&1
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/${TAG}_c1_launches.csv \
  python scripts/prof_c1.py > $O/${TAG}_c1.log 2>&1
echo profile_round done
