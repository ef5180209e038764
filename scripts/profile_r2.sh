# round-2 ncu evidence: launch list of the bench, one full capture of K1 (7B
# layer) and of the prefill attention kernel
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_pair_kernel -s 2 -c 1 \
    -o gpurun_out/r2_k1_full python scripts/k1_probe.py 4 > gpurun_out/r2_k1_full.log 2>&1
ncu -i gpurun_out/r2_k1_full.ncu-rep --page raw --csv > gpurun_out/r2_k1_full_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_k1_full.ncu-rep --page details --csv > gpurun_out/r2_k1_full_details.csv 2>/dev/null
ls -la gpurun_out | tail -20
