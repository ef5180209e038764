# A/B of the two-lane resident restore (HC_RESIDENT_STREAMS=1: one stream), interleaved
for i in 1 2; do
  for c in 1 2; do
    HC_RESIDENT_STREAMS=$c timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-recompute 2>&1 | tail -1 > gpurun_out/abr_$c.json
    python -c "import json; d=json.load(open('gpurun_out/abr_$c.json')); r=d['restore_latency_ms']; print('lanes=$c', round(r['resident'],3), round(d['roofline']['k1_ms']*32,3), d['clocks']['sm_mhz'])"
  done
done
