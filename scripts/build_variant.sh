#!/bin/bash
# build libce_gpu.so with extra nvcc defines into scripts/build/ab/<name>.so (development A/B tests)
# usage: scripts/build_variant.sh <name> [-DFOO ...]
set -e
name=$1; shift
D=/root/repo/paper_1603_09133_b200/csrc
O=/root/repo/scripts/build/ab/$name
mkdir -p $O
for f in sweep apply dense krylov; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC "$@" -c $D/$f.cu -o $O/$f.o
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -static-libstdc++ -Xcompiler -static-libgcc -Xlinker --exclude-libs,ALL -o $O.so $O/*.o $D/build/validate.o $D/build/shard.o $D/build/assemble.o $D/build/pattern.o $D/build/driver.o $D/build/capi.o $D/build/problem.o $D/build/io.o -lcudart_static -lrt -lpthread -ldl
echo built $O.so
