timeout 900 python -m pytest tests/test_serve_gpu.py -x -q -m gpu 2>&1 | tail -2
timeout 900 python scripts/serve_bench.py --skip-conv --long-sessions 0 --out gpurun_out/serve_sav.json 2>&1 | grep "^saving"
HC_SERVE_GRAPHS=0 timeout 900 python scripts/serve_bench.py --skip-conv --long-sessions 0 --out gpurun_out/serve_sav0.json 2>&1 | grep "^saving"
python - <<'PY'
import json
for f in ("gpurun_out/serve_sav.json", "gpurun_out/serve_sav0.json"):
    d = json.load(open(f))["saving"]
    print(f, {k: round(v["tbt_mean_s"] * 1e3, 3) for k, v in d.items() if isinstance(v, dict) and "tbt_mean_s" in v})
PY
