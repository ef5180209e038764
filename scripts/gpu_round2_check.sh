timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 >> gpurun_out/gputest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log > gpurun_out/bench_latest.json
