timeout 900 python -m pytest tests/test_sharded_restore_gpu.py tests/test_peer_sharded_gpu.py -q -x -m gpu 2>&1 | tail -15
timeout 1200 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/sharded_7b_2re.log 2>&1; echo rc=$?
tail -c 3500 gpurun_out/sharded_7b_2re.log
