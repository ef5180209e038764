# attention: grid of (pair, head) CTAs (HC_FA_PERSIST=0) vs the persistent kernel
# (default for a single sequence whose K/V fit in L2) vs $LIBS (alt builds)
for i in 1 2 3; do
  echo "grid:    $(HC_FA_PERSIST=0 REPS=50 timeout 120 python scripts/attn_probe.py 4096 2>&1 | tail -1)"
  echo "persist: $(REPS=50 timeout 120 python scripts/attn_probe.py 4096 2>&1 | tail -1)"
  for lib in $LIBS; do
    echo "$lib: $(HC_LIB_PATH=$lib REPS=50 timeout 120 python scripts/attn_probe.py 4096 2>&1 | tail -1)"
  done
done
