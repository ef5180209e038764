# head-sharded bench on one GPU (2 ranks = 2 processes sharing the GPU via CUDA IPC)
free -g; nproc
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/sharded_7b_2.log 2>&1; echo rc=$?
tail -c 2500 gpurun_out/sharded_7b_2.log
timeout 1200 python bench.py --gpus 2 --config llama2-70b --steps 3 --warmup 3 > gpurun_out/sharded_70b_2.log 2>&1; echo rc=$?
tail -c 2500 gpurun_out/sharded_70b_2.log
