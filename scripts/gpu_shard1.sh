timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --sharded --steps 5 --warmup 3 2>&1 | tail -3
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1
