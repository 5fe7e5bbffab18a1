#!/bin/bash
# Dev tool: link a variant of the library with one .cu replaced (and extra
# -D flags), into varlib/lib_<name>.so, for A/B timing on the GPU box.
# usage: tools/build_variant.sh <name> <variant.cu> [nvcc flags...]
set -e
name=$1; src=$2; shift 2
cd "$(dirname "$0")/.."
base=$(basename "$src" | sed 's/_var.*//; s/\.cu$//')
mkdir -p varlib
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
  --expt-relaxed-constexpr -I include -I paper_1406_5802_b200/csrc "$@" -c "$src" -o varlib/$name.o
objs=$(ls paper_1406_5802_b200/_lib/*.o | grep -v "/$base.cu.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o varlib/lib_$name.so $objs varlib/$name.o -lcudart -lpthread
rm varlib/$name.o
echo varlib/lib_$name.so
