#!/bin/bash
# Build an A/B variant of the library with extra -D flags on the L = 4096
# instantiation unit (tb_api.o and the other radial lengths are the current
# build's): tools/build_variant.sh <name> "<-DFLAGS ...>"  ->  ablibs/<name>.so
set -e
name=$1; flags=$2
cd "$(dirname "$0")/.."
mkdir -p ablibs
B=paper_1704_08364_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr \
  -DTB_L=4096 $flags -c -o /tmp/tb_inst_4096_$name.o paper_1704_08364_b200/csrc/tb_inst.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ablibs/$name.so $B/tb_api.o \
  $(ls $B/tb_inst_*.o | grep -v '_4096.o') /tmp/tb_inst_4096_$name.o
echo "ablibs/$name.so"
