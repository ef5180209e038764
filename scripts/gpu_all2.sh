timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 900 python scripts/serve_bench.py --out gpurun_out/serve_7b.json 2>&1 | grep -v "^{" | tail -12
