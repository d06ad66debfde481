# config-5 step: dynamic unit draws (default) vs the static raster, alternated on one box
for r in 1 2 3; do
  for d in 1 0; do
    B2_GEMM_DYNAMIC=$d timeout 300 python bench.py --no-ops --no-cpu --no-bf16 --steps 20 2>/dev/null | grep '^{' \
      | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('dynamic $d', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value']))"
  done
done
