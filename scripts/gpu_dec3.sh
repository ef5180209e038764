timeout 600 python -m pytest tests/test_forward_gpu.py tests/test_serve_gpu.py -x -q -m gpu 2>&1 | tail -2
cd scripts
HC_HOST_PROFILE=1 KPROF=1 B=16 CTX=512 python decode_probe.py 2>&1 | tail -30
