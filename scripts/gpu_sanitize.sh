# compute-sanitizer over the restore path's kernels (hc:: kernels only)
set -x
python scripts/sanitize_probe.py
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --kernel-name kns=2hc --print-limit 20 \
    python scripts/sanitize_probe.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
