timeout 900 python -m pytest tests/test_sharded_restore_gpu.py tests/test_cpp_facade.py -q -x -m gpu 2>&1 | tail -4
timeout 1200 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sharded_7b_2copy.log 2>&1; echo rc=$?
tail -1 gpurun_out/sharded_7b_2copy.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['restore_latency_ms'], d['speedup'], d['planner']['plan'], d['parity']['ok'])"
