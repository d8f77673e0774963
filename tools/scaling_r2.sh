# Round-2 multi-GPU evidence (one box, 4 GPUs): NCCL pipeline lockstep tests,
# then the default bench workload (configs[1] rounds, strong scaling) and the
# 7B scenario-S workload at N = 1, 2, 4 (one rank per GPU over NCCL).
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_multi.py -q -rs > gpurun_out/sc2_multi.log 2>&1
python bench.py --no-cpu-baseline --no-attn-long > gpurun_out/sc2_cfg2_n1.json 2> gpurun_out/sc2_cfg2_n1.err
for N in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N \
    bench.py --gpus $N > gpurun_out/sc2_cfg2_n$N.json 2> gpurun_out/sc2_cfg2_n$N.err
done
for N in 1 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N \
    bench.py --gpus $N --workload s7b --no-cpu-baseline --no-attn-long > gpurun_out/sc2_s7b_n$N.json 2> gpurun_out/sc2_s7b_n$N.err
done
for N in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N \
    bench.py --gpus $N --workload cfg4 --no-cpu-baseline --no-attn-long > gpurun_out/sc2_cfg4_n$N.json 2> gpurun_out/sc2_cfg4_n$N.err
done
tail -3 gpurun_out/sc2_multi.log
