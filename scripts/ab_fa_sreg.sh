# attention: scores kept in registers between the max and exponential passes
# (HC_FA_SREG=1, in-tree) vs re-read from TMEM (alt build, HC_FA_SREG=0);
# persistent (7B) and grid (16K x 40 heads) kernels, interleaved
bash scripts/build_alt.sh nosreg attention_tc.cu "-DHC_FA_SREG=0" >/dev/null
for i in 1 2 3; do
  echo "sreg   7B:  $(REPS=50 timeout 120 python scripts/attn_probe.py 4096 2>&1 | tail -1)"
  echo "nosreg 7B:  $(HC_LIB_PATH=alt_lib/libhcache_nosreg.so REPS=50 timeout 120 python scripts/attn_probe.py 4096 2>&1 | tail -1)"
  echo "sreg   grid 7B:  $(HC_FA_PERSIST=0 REPS=50 timeout 120 python scripts/attn_probe.py 4096 2>&1 | tail -1)"
  echo "nosreg grid 7B:  $(HC_FA_PERSIST=0 HC_LIB_PATH=alt_lib/libhcache_nosreg.so REPS=50 timeout 120 python scripts/attn_probe.py 4096 2>&1 | tail -1)"
done
for i in 1 2; do
  echo "sreg   16K: $(REPS=5 timeout 120 python scripts/attn_probe.py 16384 2>&1 | tail -1)"
  echo "nosreg 16K: $(HC_LIB_PATH=alt_lib/libhcache_nosreg.so REPS=5 timeout 120 python scripts/attn_probe.py 16384 2>&1 | tail -1)"
done
