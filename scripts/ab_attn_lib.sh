# attention A/B: in-tree library vs alt builds ($LIBS), interleaved, 7B layer shape
for i in 1 2 3; do
  for lib in paper_2410_05004_b200/lib/libhcache_b200.so $LIBS; do
    echo "$lib: $(HC_LIB_PATH=$lib REPS=50 timeout 120 python scripts/attn_probe.py 4096 2>&1 | tail -1)"
  done
done
