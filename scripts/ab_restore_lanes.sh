# restore K1 lanes A/B (HC_RESTORE_LANES=1/2): 7B e2e + timeline, long-context serving TTFT
for i in 1 2; do
  for l in 1 2; do
    HC_RESTORE_LANES=$l timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/rl_$l.json
    python -c "import json; d=json.load(open('gpurun_out/rl_$l.json')); print('lanes=$l', d['planner']['plan'], 'e2e', round(d['restore_latency_ms']['e2e'],2), 'tl', round(d['timeline']['total_ms'],2), d['clocks']['sm_mhz'])"
  done
done
for l in 1 2; do
  HC_RESTORE_LANES=$l timeout 900 python scripts/serve_bench.py --skip-conv --skip-saving --strategies HCACHE --out gpurun_out/lcl_$l.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/lcl_$l.json')); lc=d['long_context']; h=lc['strategies']['HCACHE']
print('serve lanes=$l', lc['plan'], 'p50 %.1f p95 %.1f'%(h['ttft_p50_s']*1e3,h['ttft_p95_s']*1e3), [r[1] for r in h['per_request']])"
done
