timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
cd scripts; KPROF=1 B=16 CTX=512 python decode_probe.py 2>&1 | grep -v Warn | tail -14
cd ..; timeout 900 python scripts/serve_bench.py --out gpurun_out/serve_7b.json 2>&1 | grep -v "^{" | tail -9
