python scripts/scatter_probe.py
ncu --set full --clock-control none -k regex:kv_scatter -s 5 -c 1 -o gpurun_out/k4_scatter_r1c python scripts/scatter_probe.py > gpurun_out/k4_scatter_r1c.log 2>&1
