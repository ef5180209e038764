ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_r1b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_pair_kernel -s 40 -c 1 -o gpurun_out/k1_pair_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-recompute > gpurun_out/k1_pair_full.log 2>&1
ls gpurun_out/
