timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/mg60.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --no-attn-long > gpurun_out/mg60_n2.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 --no-attn-long > gpurun_out/mg60_n4.json 2>/dev/null
