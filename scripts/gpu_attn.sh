timeout 600 python -m pytest tests/test_k6_blocks_gpu.py -x -q -m gpu -k attention 2>&1 | tail -15
timeout 600 python -m pytest tests/test_recompute_gpu.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python scripts/prof_k6.py
