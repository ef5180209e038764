# planner profile warm-up A/B (HC_PROFILE_WARM_S): plan and e2e of 13B and 7B
for c in llama2-13b llama2-7b; do
  for w in 0.2 1.0; do
    HC_PROFILE_WARM_S=$w timeout 900 python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/warm_${c}_$w.json
    python -c "import json; d=json.load(open('gpurun_out/warm_${c}_$w.json')); print('$c warm=$w', d['planner']['plan'], round(d['planner']['predicted_ms'],2), 'e2e', round(d['restore_latency_ms']['e2e'],2), 'tl', round(d['timeline']['total_ms'],2), d['clocks']['sm_mhz'], d['planner']['profiled'])"
  done
done
