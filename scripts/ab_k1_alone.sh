# K1 alone (k1_probe, 200 launches) in-tree vs $LIBS, interleaved x4
for i in 1 2 3 4; do
  for lib in paper_2410_05004_b200/lib/libhcache_b200.so $LIBS; do
    echo "$lib: $(HC_LIB_PATH=$lib timeout 120 python scripts/k1_probe.py 200 2>&1 | tail -1)"
  done
done
