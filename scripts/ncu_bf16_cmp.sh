# ncu --set full: our bf16 GEMM vs cuBLAS's at the config-5 shape (65536 x 4096 x 4096)
ncu --set full --clock-control none -k regex:k_gemm_tc --launch-skip 1 -c 1 -o gpurun_out/bf16_ours -f python scripts/gemm_bf16_one.py 4096 65536 > gpurun_out/bf16_ours.log 2>&1
ncu --set full --clock-control none -k regex:nvjet --launch-skip 1 -c 1 -o gpurun_out/bf16_cublas -f python scripts/cublas_bf16_one.py > gpurun_out/bf16_cublas.log 2>&1
