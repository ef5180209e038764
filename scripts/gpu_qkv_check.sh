timeout 900 python -m pytest tests/test_recompute_gpu.py tests/test_recompute_7b_gpu.py tests/test_restore_gpu.py tests/test_serve_gpu.py tests/test_forward_gpu.py -q -x -m gpu 2>&1 | tail -5
for i in 1 2; do
HC_QKV_SPLIT=1 timeout 300 python scripts/k6_breakdown.py --out gpurun_out/k6_split.json 2>&1 | tail -1
timeout 300 python scripts/k6_breakdown.py --out gpurun_out/k6_fused.json 2>&1 | tail -1
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fused.log 2>&1; tail -1 gpurun_out/bench_fused.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['restore_latency_ms'], d['planner']['plan'], d['planner']['profiled'], d['parity']['ok'], d['clocks'])"
