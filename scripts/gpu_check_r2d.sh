timeout 300 python scripts/zero_copy_probe.py 2>&1 | tail -8
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_7b_strict.log 2>&1
tail -1 gpurun_out/bench_7b_strict.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['restore_latency_ms'], d['strict_plan'], d['parity']['ok'])"
timeout 1500 python bench.py --config opt-30b --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_30b_e2e.log 2>&1
tail -1 gpurun_out/bench_30b_e2e.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['restore_latency_ms'], d['e2e'])"
