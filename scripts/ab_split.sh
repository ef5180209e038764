# A/B of the token split of the first hidden layer (HC_SPLIT=1 enables it), interleaved
for i in 1 2; do
  for c in 1 0; do
    if [ $c = 1 ]; then unset HC_SPLIT; else export HC_SPLIT=1; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/abs_$c.json
    python -c "import json; d=json.load(open('gpurun_out/abs_$c.json')); r=d['restore_latency_ms']; p=d['planner']; print('nosplit=$c', round(r['e2e'],3), p['plan'], p['split_tokens'], round(p['predicted_ms'],3), round(p['predicted_with_split_ms'],3), round(d['timeline']['total_ms'],3), d['clocks']['sm_mhz'])"
  done
done
