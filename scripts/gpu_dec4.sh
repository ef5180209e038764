timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
cd scripts
KPROF=1 B=16 CTX=512 python decode_probe.py 2>&1 | grep -v Warn | tail -14
B=1 CTX=512 python decode_probe.py 2>&1 | tail -1
cd ..
python bench.py --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_latest.json
python -c "import json; d=json.load(open('gpurun_out/bench_latest.json')); print(d['value'], d['restore_latency_ms'], d['e2e']['value'], d['roofline']['frac'])"
