# attention A/B: in-tree library vs $ALT_LIB (interleaved), then the parity tests
for i in 1 2 3; do
  for lib in paper_2410_05004_b200/lib/libhcache_b200.so $ALT_LIB; do
    echo "$lib: $(HC_LIB_PATH=$lib timeout 120 python scripts/attn_probe.py 2>&1 | tr '\n' ' ')"
  done
done
timeout 900 python -m pytest tests/test_k6_blocks_gpu.py tests/test_recompute_gpu.py tests/test_forward_gpu.py -q -x 2>&1 | tail -2
