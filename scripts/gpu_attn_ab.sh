echo base; HC_LIB_PATH=$PWD/scripts/_base/lib_base.so python scripts/attn_probe.py
echo new; python scripts/attn_probe.py
timeout 900 python scripts/serve_bench.py --skip-conv --skip-saving --strategies HCACHE --out gpurun_out/serve_long.json 2>&1 | grep -v "^{" | tail -3
python -c "
import json; d=json.load(open('gpurun_out/serve_long.json'))
for k,v in d['long_context']['strategies'].items(): print(k, v['per_request'])
"
