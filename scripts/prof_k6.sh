python scripts/prof_k6.py
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_gemm|attn|row_stats|embed" -s 40 -c 14 --csv --log-file gpurun_out/k6_launches.csv python scripts/prof_k6.py > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/k6_launches.csv')))
h = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
hdr = rows[h]
for r in rows[h+1:]:
    print(r[hdr.index('Metric Value')], r[hdr.index('Grid Size')], r[hdr.index('Kernel Name')][:90])
PY
