#!/bin/bash
# Full library build with extra nvcc/g++ defines into scripts/build/ab/<name>.so (A/B tests)
# usage: scripts/build_ab_full.sh <name> [-DFOO ...]
set -e
name=$1; shift
D=/root/repo/paper_1603_09133_b200/csrc
O=/tmp/ab_build/$name  # objects outside the repo (gpurun ships the repo)
SO=/root/repo/scripts/build/ab/$name.so
mkdir -p $O /root/repo/scripts/build/ab
for f in $(sed -n "s/^CU := //p" $D/Makefile | sed "s/\.cu//g"); do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC "$@" -c $D/$f.cu -o $O/$f.o &
done
for f in driver capi problem io; do
  g++ -O2 -std=c++17 -fPIC -fno-fast-math -ffp-contract=off -I/usr/local/cuda/include "$@" -c $D/$f.cpp -o $O/$f.o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -static-libstdc++ -Xcompiler -static-libgcc -Xlinker --exclude-libs,ALL -o $SO $O/*.o -lcudart_static -lrt -lpthread -ldl
echo built $SO
