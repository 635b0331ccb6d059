#!/bin/bash
# Full library variant (every radial length) with extra -D flags:
# tools/build_full_variant.sh <name> "<-DFLAGS>"  ->  ablibs/<name>.so
set -e
name=$1; flags=$2
cd "$(dirname "$0")/.."
B=/tmp/tbvar_$name; mkdir -p $B ablibs
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr"
$NV $flags -c -o $B/tb_api.o paper_1704_08364_b200/csrc/tb_api.cu &
for l in 4 8 16 32 64 128 256 512 1024 2048 4096 8192 16384; do
  $NV $flags -DTB_L=$l -c -o $B/tb_inst_$l.o paper_1704_08364_b200/csrc/tb_inst.cu &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ablibs/$name.so $B/*.o
echo ablibs/$name.so
