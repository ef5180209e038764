timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_serve_gpu.py tests/test_recompute_gpu.py -x -q -m gpu 2>&1 | tail -3
cd scripts; KPROF=1 B=16 CTX=512 python decode_probe.py 2>&1 | grep -v Warn | tail -16
B=1 CTX=512 python decode_probe.py 2>&1 | tail -1
B=32 CTX=1024 python decode_probe.py 2>&1 | tail -1
