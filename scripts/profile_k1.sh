# ncu evidence for the dominant kernel (K1): launch list + one full capture
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_restore_kv -s 40 -c 1 \
    -o gpurun_out/k1_full_r1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/k1_full.log 2>&1
ls -la gpurun_out
