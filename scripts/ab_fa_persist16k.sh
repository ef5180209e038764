for i in 1 2; do
  echo "grid 16K:        $(REPS=5 timeout 120 python scripts/attn_probe.py 16384 2>&1 | tail -1)"
  echo "persist hm 16K:  $(HC_FA_PERSIST=2 REPS=5 timeout 120 python scripts/attn_probe.py 16384 2>&1 | tail -1)"
  echo "persist rm 16K:  $(HC_FA_PERSIST=1 REPS=5 timeout 120 python scripts/attn_probe.py 16384 2>&1 | tail -1)"
done
