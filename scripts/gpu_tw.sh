timeout 600 python -m pytest tests/test_restore_gpu.py -x -q -m gpu -k "token_wise" 2>&1 | tail -15
