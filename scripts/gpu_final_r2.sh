# round-2 final evidence: GPU tests, smoke, bench (N=1), ncu launch list of the bench
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 >> gpurun_out/gputest_final.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final.log 2>&1
tail -1 gpurun_out/bench_final.log > gpurun_out/bench_final.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r2_final_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_final_launches_bench.log 2>&1
cat gpurun_out/gputest_final.log
