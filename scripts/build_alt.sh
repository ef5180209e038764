#!/bin/bash
# Alternative library build for A/B runs: one .cu recompiled with extra
# defines, linked with the in-tree objects of everything else.
#   scripts/build_alt.sh NAME SRC.cu "-DFOO=1 ..."   -> alt_lib/libhcache_NAME.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2410_05004_b200/csrc
OBJ=$ROOT/paper_2410_05004_b200/build_obj
mkdir -p $ROOT/alt_lib
base=$(basename $2 .cu)
/usr/local/cuda/bin/nvcc -ccbin g++ -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC --expt-relaxed-constexpr $3 -c $CS/$2 -o /tmp/alt_$1_$base.o
/usr/local/cuda/bin/nvcc -ccbin g++ -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o $ROOT/alt_lib/libhcache_$1.so /tmp/alt_$1_$base.o $(ls $OBJ/*.o | grep -v "/$base.cu.o") -lpthread -ldl -lrt
echo built alt_lib/libhcache_$1.so
