set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/ev_n1.json 2> gpurun_out/ev_n1.err
python bench.py --impl reference > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/ev_n2.json 2> gpurun_out/ev_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > gpurun_out/ev_n4.json 2> gpurun_out/ev_n4.err
CUDA_VISIBLE_DEVICES=0 bash tools/profile_ncu.sh
