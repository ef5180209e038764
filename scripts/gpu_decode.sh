cd scripts
B=16 CTX=512 python decode_probe.py
B=1 CTX=512 python decode_probe.py
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
tot = sum(v[1] for v in agg.values())
print('total ns', tot, 'launches', sum(v[0] for v in agg.values()))
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{v[1]/1e3:10.1f} us {v[0]:5d} {k}")
PY
