# BASELINE configs 3-5 at N=1 with the round-2 code, then the ncu launch list
# of the 7B bench restricted to the restore path's kernels (setup fills skipped)
for c in llama2-13b opt-30b llama2-70b; do
  timeout 1500 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$c.json
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', d['value'], d['restore_latency_ms'], d['e2e']['value'], d.get('planner',{}).get('plan'), d['roofline']['frac'], d['clocks']['sm_mhz'], d.get('parity',{}).get('ok'))" 2>&1 | tail -2
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"tc_gemm|attn_fa|row_stats|center_rows|kv_scatter|zero_i32|embed|gather_stats" -c 4000 --csv \
    --log-file gpurun_out/r2_final_launches_restore.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_final_launches_restore.log 2>&1
echo ncu rc=$?
