# config-5 step with the collectives' SM reserve at 0 / 8 / 16 (1-rank NCCL
# communicator: the reserve's cost on the GEMMs, no real collectives)
for r in 1 2; do
for gb in 65536 8192; do
for v in 0 8 16; do
  B2_FORCE_NCCL=1 B2_COMM_SMS=$v timeout 300 python bench.py --no-ops --no-cpu --no-bf16 --steps 10 --global-batch $gb 2>/dev/null \
    | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('gb $gb reserve $v', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])"
done; done; done
