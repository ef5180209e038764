# attention: share of exp2 pairs on the FMA pipe (HC_FA_EMU, compile time) -- default lib (3) vs alt builds
for i in 1 2; do
  for lib in ${LIBS:-paper_2410_05004_b200/lib/libhcache_b200.so alt_lib/libhcache_emu2.so alt_lib/libhcache_emu4.so}; do
    echo "$lib: $(HC_LIB_PATH=$lib timeout 120 python scripts/attn_probe.py 2>&1 | tr '\n' ' ')"
  done
done
