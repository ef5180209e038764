# one ncu --set full capture of the prefill attention kernel (7B layer: n=4096, 32 heads, dense)
ncu --set full --clock-control none --import-source on -k regex:attn_ -s 3 -c 1 -o gpurun_out/attn_full python scripts/attn_probe.py 4096 > gpurun_out/attn_full.log 2>&1
ls -la gpurun_out/attn_full*
