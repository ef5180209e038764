free -g | head -2
timeout 1500 python scripts/serve_bench.py --out gpurun_out/serve_7b.json 2>&1 | grep -v "^{" | tail -22
