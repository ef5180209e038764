# round-2 (late) evidence for the current build: K6 per-kernel breakdown at
# the power-capped clock, one ncu --set full capture of K1 (traffic) and of
# the prefill attention
set -x
timeout 300 python scripts/k6_breakdown.py > gpurun_out/k6_breakdown.log 2>&1
tail -40 gpurun_out/k6_breakdown.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_pair_kernel -s 2 -c 1 \
    -o gpurun_out/r2c_k1_full python scripts/k1_probe.py 4 > gpurun_out/r2c_k1_full.log 2>&1
ncu -i gpurun_out/r2c_k1_full.ncu-rep --page raw --csv > gpurun_out/r2c_k1_full_raw.csv 2>/dev/null
ncu -i gpurun_out/r2c_k1_full.ncu-rep --page details --csv > gpurun_out/r2c_k1_full_details.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fa -s 4 -c 1 \
    -o gpurun_out/r2c_attn python scripts/prof_k6.py > gpurun_out/r2c_attn.log 2>&1
ncu -i gpurun_out/r2c_attn.ncu-rep --page raw --csv > gpurun_out/r2c_attn_raw.csv 2>/dev/null
ncu -i gpurun_out/r2c_attn.ncu-rep --page details --csv > gpurun_out/r2c_attn_details.csv 2>/dev/null
ls -la gpurun_out | tail -20
