# r1c ncu evidence: bench launch list, K1 pair kernel (--set full), two-Q-tile attention (--set full)
ncu --metrics gpu__time_duration.sum --clock-control none -s 500 -c 400 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_r1c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_pair_kernel -s 40 -c 1 -o gpurun_out/k1_pair_r1c python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-recompute > gpurun_out/k1_pair_r1c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fa -s 3 -c 1 -o gpurun_out/attn_fa_r1c python scripts/attn_probe.py 4096 > gpurun_out/attn_fa_r1c.log 2>&1
ls gpurun_out/
