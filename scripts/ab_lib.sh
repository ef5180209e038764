# resident / K1 A/B between the in-tree library and an alternative build ($ALT_LIB), interleaved
for i in 1 2 3; do
  for lib in paper_2410_05004_b200/lib/libhcache_b200.so $ALT_LIB; do
    echo -n "$lib: "; HC_LIB_PATH=$lib python scripts/resident_probe.py 2>&1 | tail -1
  done
done
