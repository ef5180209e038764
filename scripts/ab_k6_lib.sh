# K6 layer span (k6_breakdown) in-tree vs $LIBS, interleaved
for i in 1 2 3; do
  for lib in paper_2410_05004_b200/lib/libhcache_b200.so $LIBS; do
    echo "$lib: $(HC_LIB_PATH=$lib timeout 300 python scripts/k6_breakdown.py --out gpurun_out/k6_ab.json 2>&1 | tail -1)"
  done
done
