cd scripts
echo default; python gemm_probe.py
echo split; HC_GEMM_SPLIT=1 python gemm_probe.py
cd ..
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
cd scripts; KPROF=1 B=16 CTX=512 python decode_probe.py 2>&1 | grep -v Warn | tail -14
