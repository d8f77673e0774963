#!/bin/bash
# f1 ablation evidence (tools/ablation.py) at P=1 and P=4 (torchrun, NCCL)
mkdir -p gpurun_out
python tools/ablation.py > gpurun_out/abl_p1.json 2> gpurun_out/abl_p1.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 \
    tools/ablation.py > gpurun_out/abl_p4.json 2> gpurun_out/abl_p4.err
