# attention: share of exp2 pairs on the FMA pipe (HC_FA_EMU, compile time) -- in-tree lib vs alt builds.
# Build an alt library (N = pairs of every 8 on the FMA pipe), from paper_2410_05004_b200/csrc:
#   nvcc -ccbin g++ -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
#     --expt-relaxed-constexpr -DHC_FA_EMU=N -c attention_tc.cu -o /tmp/attn_emuN.o
#   nvcc -ccbin g++ -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
#     -o ../../alt_lib/libhcache_emuN.so /tmp/attn_emuN.o $(ls ../build_obj/*.o | grep -v attention_tc) \
#     -lpthread -ldl -lrt
for i in 1 2; do
  for lib in ${LIBS:-paper_2410_05004_b200/lib/libhcache_b200.so alt_lib/libhcache_emu2.so alt_lib/libhcache_emu4.so}; do
    echo "$lib: $(HC_LIB_PATH=$lib timeout 120 python scripts/attn_probe.py 2>&1 | tr '\n' ' ')"
  done
done
