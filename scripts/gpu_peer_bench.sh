export HC_DIST_BACKEND=gloo HC_FORCE_DEVICE=0
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 3 --warmup 3 2>&1 | grep -v Warning | tail -4 | cut -c1-1200
unset HC_DIST_BACKEND HC_FORCE_DEVICE
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 1 --sharded --steps 5 --warmup 3 2>&1 | grep -v Warning | tail -2 | cut -c1-1500
