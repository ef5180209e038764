# memcheck / racecheck over the head-sharded restore (2 processes on the GPU,
# IPC-mapped peer slots, flags, the fused multi-source K1, the replicated prefix)
for tool in memcheck racecheck; do
  timeout 1800 compute-sanitizer --tool $tool --target-processes all --kernel-name kns=2hc --print-limit 20 \
    python -m pytest tests/test_sharded_restore_gpu.py -q -x -m gpu -k "bit_exact and 700 or recompute_prefix and 640" \
    > gpurun_out/sanitize_sharded_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_sharded_$tool.log | sort | uniq -c
done
