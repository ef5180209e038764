timeout 600 python -m pytest tests/test_forward_gpu.py tests/test_serve_gpu.py tests/test_recompute_gpu.py -x -q -m gpu 2>&1 | tail -4
cd scripts
B=16 CTX=512 python decode_probe.py
B=1 CTX=512 python decode_probe.py
B=16 CTX=2048 python decode_probe.py
B=16 CTX=512 REPS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ../gpurun_out/decode_launches.csv python decode_probe.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(l for l in open('../gpurun_out/decode_launches.csv') if l.startswith('"')))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r['Metric Name'] != 'gpu__time_duration.sum': continue
    k = r['Kernel Name'][:60]
    agg[k][0] += 1
    agg[k][1] += float(r['Metric Value'].replace(',', ''))
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{v[1]/4e3:10.1f} us/step {v[0]:5d} {k}")
PY
