# ncu --set full of K1 (7B layer) with the final round-2 build (roofline.traffic)
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_pair_kernel -s 2 -c 1 \
    -o gpurun_out/r2e_k1_full python scripts/k1_probe.py 4 > gpurun_out/r2e_k1_full.log 2>&1
ncu -i gpurun_out/r2e_k1_full.ncu-rep --page raw --csv > gpurun_out/r2e_k1_full_raw.csv 2>/dev/null
ncu -i gpurun_out/r2e_k1_full.ncu-rep --page details --csv > gpurun_out/r2e_k1_full_details.csv 2>/dev/null
