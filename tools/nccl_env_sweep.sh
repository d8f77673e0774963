# ms per tick of the 7B scenario-S workload at N ranks under NCCL protocol settings
N=${1:-2}
for E in "X=1" "NCCL_PROTO=LL" "NCCL_PROTO=LL128" "NCCL_PROTO=Simple" "NCCL_MAX_NCHANNELS=2" "NCCL_NVLS_ENABLE=0"; do
  env $E python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$((RANDOM % 800 + 100)) \
    bench.py --gpus $N --workload s7b --no-cpu-baseline --no-attn-long --no-profile 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$E', d['ms_per_step'], d['value'])"
done
