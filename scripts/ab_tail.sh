# tail split of the last wave at K=4096 (HC_TAIL_MIN_KB=32 alt build) vs K >= 96 k-blocks only
for i in 1 2; do
  for lib in paper_2410_05004_b200/lib/libhcache_b200.so alt_lib/libhcache_tail32.so; do
    echo "== $lib"; HC_LIB_PATH=$lib HC_GEMM_SPLIT=1 python scripts/gemm_k6_probe.py | head -1
    echo "k6: $(HC_LIB_PATH=$lib timeout 300 python scripts/k6_breakdown.py --out gpurun_out/k6_tail.json 2>&1 | tail -1)"
  done
done
