for ar in 1 4; do
timeout 900 python scripts/serve_bench.py --skip-conv --skip-saving --arenas $ar --strategies HCACHE,KV_OFFLOAD --out gpurun_out/serve_long_a$ar.json 2>&1 | grep -v "^{" | tail -5
python -c "
import json; d=json.load(open('gpurun_out/serve_long_a$ar.json'))
print('arenas $ar plan', d['long_context']['plan'])
for k,v in d['long_context']['strategies'].items(): print(k, v['per_request'])
"
done
