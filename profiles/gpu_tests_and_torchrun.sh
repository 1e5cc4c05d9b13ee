timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
# the torchrun launch path of bench.py (world 1: NCCL init, all-reduce of totals, max over ranks)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 1 --instructions 2000000 --no-cpu-baseline 2>&1 | tail -2
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 1 --warmup 1 2>&1 | tail -1
