# memcheck / racecheck after the register-resident softmax chunks and the
# direct D2H save path: the restore probe (single GPU) and the device range
# snapshots (direct path into chunk slots)
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --kernel-name kns=2hc --print-limit 20 \
    python scripts/sanitize_probe.py > gpurun_out/sanitize4_$tool.log 2>&1
  echo "probe $tool rc=$?"; tail -2 gpurun_out/sanitize4_$tool.log
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 \
  python -m pytest -q -x tests/test_restore_gpu.py -k "snapshot" > gpurun_out/sanitize4_snapshot.log 2>&1
echo "snapshot memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize4_snapshot.log | sort | uniq -c
