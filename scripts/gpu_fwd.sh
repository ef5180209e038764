timeout 600 python -m pytest tests/test_forward_gpu.py tests/test_recompute_gpu.py tests/test_k6_blocks_gpu.py -x -q -m gpu 2>&1 | tail -15
