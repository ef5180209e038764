timeout 600 python -m pytest tests/test_serve_gpu.py tests/test_forward_gpu.py -x -q -m gpu 2>&1 | tail -30
