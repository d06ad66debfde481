timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
for i in 1 2; do
python bench.py --no-ops --no-cpu --no-bf16 --steps 20 > gpurun_out/ab_L$i.json 2>/dev/null
B2_LAZY_FP32=0 python bench.py --no-ops --no-cpu --no-bf16 --steps 20 > gpurun_out/ab_E$i.json 2>/dev/null
done
