nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_k1_gpu.py -x -q -m gpu 2>&1 | tail -40
