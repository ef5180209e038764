# BASELINE configs 2-5 at N=1, one JSON line each (gpurun_out/bench_<config>.json)
for c in llama2-7b llama2-13b opt-30b llama2-70b; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_$c.json
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', d['value'], d['restore_latency_ms'], d['e2e']['value'], d.get('planner',{}).get('plan'), d['roofline']['frac'], d['clocks']['sm_mhz'])" 2>&1 | tail -2
done
