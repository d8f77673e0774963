# Round-2 multi-GPU evidence (one box, 4 GPUs): NCCL pipeline lockstep tests,
# then the default bench workload (configs[1] rounds, strong scaling), the 7B
# and 13B scenario-S workloads and configs[4] (72B) at N = 1, 2, 4 (one rank
# per GPU over NCCL), and the f1 ablation at P = 4.
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_multi.py -q -rs > gpurun_out/sc5_multi.log 2>&1
for W in cfg2 s7b cfg4 cfg5; do
  for N in 1 2 4; do
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$N$((RANDOM % 90 + 10)) \
      bench.py --gpus $N --workload $W --no-cpu-baseline --no-attn-long > gpurun_out/sc5_${W}_n$N.json 2> gpurun_out/sc5_${W}_n$N.err
  done
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29471 \
  tools/ablation.py > gpurun_out/sc5_ablation_p4.json 2> gpurun_out/sc5_ablation_p4.err
tail -3 gpurun_out/sc5_multi.log
