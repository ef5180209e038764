# planner profile with 4-layer recompute calls: plan, profiled costs and e2e for 7B and 13B (two runs each)
for c in llama2-7b llama2-13b; do
  for i in 1 2; do
    timeout 900 python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/apl_${c}_$i.json
    python -c "import json; d=json.load(open('gpurun_out/apl_${c}_$i.json')); print('$c', d['planner']['plan'], round(d['planner']['predicted_ms'],2), 'e2e', round(d['restore_latency_ms']['e2e'],2), 'tl', round(d['timeline']['total_ms'],2), d['clocks']['sm_mhz'], {k: round(v,4) for k,v in d['planner']['profiled'].items()})"
  done
done
