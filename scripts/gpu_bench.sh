timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_latest.json
python -c "import json; d=json.load(open('gpurun_out/bench_latest.json')); print(d['value'], d['restore_latency_ms'], d['e2e']['value'], d['planner']['plan'], d['roofline']['frac'], d['clocks'])"
