# decode step: split-K epilogue and split-KV decode attention launched with
# PDL (in-tree) vs plain launches (ab_lib/libhcache_nopdl_dec.so, built in
# the container by scripts/build_ab_decode_pdl.sh from the previous commit's
# two files), interleaved; B sequences x 1 token, 7B shape
for i in 1 2 3; do
  for B in 1 16; do
    echo "pdl   B=$B: $(B=$B CTX=512 REPS=30 timeout 300 python scripts/decode_probe.py 2>&1 | tail -1)"
    echo "plain B=$B: $(HC_LIB_PATH=ab_lib/libhcache_nopdl_dec.so B=$B CTX=512 REPS=30 timeout 300 python scripts/decode_probe.py 2>&1 | tail -1)"
  done
done
