# ncu --set full of the persistent attention kernel (7B layer) after the register-resident score chunks
ncu --set full --clock-control none --import-source on -k regex:attn_fa_persist -s 3 -c 1 \
    -o gpurun_out/r2f_attn_persist python scripts/attn_probe.py 4096 > gpurun_out/r2f_attn_persist.log 2>&1
ncu -i gpurun_out/r2f_attn_persist.ncu-rep --page raw --csv > gpurun_out/r2f_attn_persist_raw.csv 2>/dev/null
ncu -i gpurun_out/r2f_attn_persist.ncu-rep --page details --csv > gpurun_out/r2f_attn_persist_details.csv 2>/dev/null
tail -3 gpurun_out/r2f_attn_persist.log
