# attention: per-(pair, head) CTAs (default) vs one persistent CTA per SM (HC_FA_PERSIST=1)
HC_FA_PERSIST=1 timeout 120 python scripts/attn_probe.py 1024 2>&1 | tail -2
for i in 1 2 3; do
  echo "grid:    $(REPS=50 timeout 120 python scripts/attn_probe.py 4096 2>&1 | tail -1)"
  echo "persist: $(HC_FA_PERSIST=1 REPS=50 timeout 120 python scripts/attn_probe.py 4096 2>&1 | tail -1)"
done
echo "grid 16K:    $(REPS=5 timeout 120 python scripts/attn_probe.py 16384 2>&1 | tail -1)"
echo "persist 16K: $(HC_FA_PERSIST=1 REPS=5 timeout 120 python scripts/attn_probe.py 16384 2>&1 | tail -1)"
HC_FA_PERSIST=1 timeout 600 python -m pytest tests/test_k6_blocks_gpu.py tests/test_stale_pages_gpu.py tests/test_recompute_gpu.py -q -x -m gpu 2>&1 | tail -3
