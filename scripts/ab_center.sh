# A/B of the LayerNorm centering guard (HC_LN_CENTER=0 disables it), interleaved
for i in 1 2; do
  for c in 0 1; do
    HC_LN_CENTER=$c timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-recompute 2>&1 | tail -1 > gpurun_out/ab_$c.json
    python -c "import json; d=json.load(open('gpurun_out/ab_$c.json')); r=d['restore_latency_ms']; print('center=$c', round(r['resident'],3), round(r['e2e'],3), round(d['roofline']['k1_ms']*32,3), d['clocks']['sm_mhz'])"
  done
done
