# K1 / resident A/B between the in-tree library and alt builds ($LIBS), interleaved
for i in 1 2 3; do
  for lib in paper_2410_05004_b200/lib/libhcache_b200.so $LIBS; do
    echo "$lib: $(HC_LIB_PATH=$lib timeout 120 python scripts/k1_probe.py 200 2>&1 | tail -1) | $(HC_LIB_PATH=$lib timeout 120 python scripts/resident_probe.py 2>&1 | tail -1)"
  done
done
