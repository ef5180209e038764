timeout 900 python -m pytest tests/test_recompute_gpu.py tests/test_k6_blocks_gpu.py -q -m gpu -s 2>&1 | grep -E "assert|passed|failed|Error|recompute max" | head -30
