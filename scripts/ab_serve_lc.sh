# long-context serving TTFT, repeated: K1 lanes 2 (default) vs 1 (HC_RESIDENT_STREAMS=1)
for i in 1 2; do
  for l in 0 1; do
    if [ $l = 1 ]; then export HC_RESIDENT_STREAMS=1; else unset HC_RESIDENT_STREAMS; fi
    timeout 900 python scripts/serve_bench.py --skip-conv --skip-saving --strategies HCACHE --out gpurun_out/lc_$l_$i.json > /dev/null 2>&1
    python -c "
import json; d=json.load(open('gpurun_out/lc_$l_$i.json')); lc=d['long_context']; h=lc['strategies']['HCACHE']
print('lanes_env=$l', lc['plan'], 'p50 %.1f p95 %.1f'%(h['ttft_p50_s']*1e3,h['ttft_p95_s']*1e3), [r[1] for r in h['per_request']])"
  done
done
unset HC_RESIDENT_STREAMS
