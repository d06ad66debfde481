# ncu --set full of one K=1000 C-store GEMM launch: abtest_old/ tree vs the working tree
NCU="ncu --set full --clock-control none -k regex:k_gemm_tc --launch-skip 2 -c 1"
(cd abtest_old && $NCU -o ../gpurun_out/ab_old -f python scripts/epi_matrix.py 1000 > ../gpurun_out/ab_old.log 2>&1)
$NCU -o gpurun_out/ab_new -f python scripts/epi_matrix.py 1000 > gpurun_out/ab_new.log 2>&1
