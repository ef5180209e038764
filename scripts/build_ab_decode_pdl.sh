# builds ab_lib/libhcache_nopdl_dec.so HERE (needs git; run before gpurun)
set -e
OBJ=paper_2410_05004_b200/build_obj
mkdir -p ab_lib /tmp/abdp
for f in k1_restore_kv attention; do
  git show HEAD:paper_2410_05004_b200/csrc/$f.cu > paper_2410_05004_b200/csrc/_ab_$f.cu
  /usr/local/cuda/bin/nvcc -ccbin g++ -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC --expt-relaxed-constexpr -c paper_2410_05004_b200/csrc/_ab_$f.cu -o /tmp/abdp/$f.o
  rm paper_2410_05004_b200/csrc/_ab_$f.cu
done
/usr/local/cuda/bin/nvcc -ccbin g++ -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o ab_lib/libhcache_nopdl_dec.so /tmp/abdp/*.o \
  $(ls $OBJ/*.o | grep -v "/k1_restore_kv.cu.o" | grep -v "/attention.cu.o") -lpthread -ldl -lrt
