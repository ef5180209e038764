# long-context serving TTFT: side-stream statistics (default) vs serial (HC_RESTORE_SIDE=0)
for i in 1 2; do
  for sd in 0 1; do
    HC_RESTORE_SIDE=$sd timeout 900 python scripts/serve_bench.py --skip-conv --skip-saving --strategies HCACHE --out gpurun_out/lcs_${sd}_$i.json > /dev/null 2>&1
    python -c "
import json; d=json.load(open('gpurun_out/lcs_${sd}_$i.json')); lc=d['long_context']; h=lc['strategies']['HCACHE']
print('side=$sd', lc['plan'], 'p50 %.1f p95 %.1f'%(h['ttft_p50_s']*1e3,h['ttft_p95_s']*1e3), [r[1] for r in h['per_request']])"
  done
done
