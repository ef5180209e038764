timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
HC_DUMP_TIMELINE=gpurun_out/timeline.txt timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_latest.json
python -c "import json; d=json.load(open('gpurun_out/bench_latest.json')); print(d['value'], d['restore_latency_ms'], d['speedup'], d['planner'], d['timeline'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
