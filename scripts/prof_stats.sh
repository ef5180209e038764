ncu --set full --clock-control none -k regex:row_stats -s 5 -c 1 -o gpurun_out/stats_full python scripts/stats_probe.py > gpurun_out/stats_full.log 2>&1
python scripts/stats_probe.py
