# 4 ranks sharing the box's one GPU (functional multi-rank runs; PCIe and SMs are shared)
timeout 1500 python bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/sharded_7b_4.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/sharded_7b_4.log
timeout 1500 python bench.py --gpus 4 --config llama2-70b --steps 3 --warmup 3 > gpurun_out/sharded_70b_4.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/sharded_70b_4.log
