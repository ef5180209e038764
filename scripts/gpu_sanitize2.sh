# initcheck needs every writer instrumented (torch's kernels write the page
# tables and inputs the hc kernels read), so no kernel filter here
timeout 1800 compute-sanitizer --tool initcheck --print-limit 20 python scripts/sanitize_probe.py > gpurun_out/sanitize_initcheck_all.log 2>&1
echo "initcheck rc=$?"; grep -E "ERROR SUMMARY|sanitize probe" gpurun_out/sanitize_initcheck_all.log
grep -A4 "Uninitialized" gpurun_out/sanitize_initcheck_all.log | grep "Device Frame" | sort | uniq -c | sort -rn | head -10
