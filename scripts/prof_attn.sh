ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 2 -c 1 -o gpurun_out/attn_full python scripts/prof_k6.py > gpurun_out/attn_full.log 2>&1
ls -la gpurun_out/attn_full*
