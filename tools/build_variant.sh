#!/bin/bash
# Build libdecdec.so from a git revision into build/libdecdec_<name>.so (A/B timing with DECDEC_LIB).
# usage: bash tools/build_variant.sh <rev> <name> ["-DMACRO=1 ..."]
set -e
rev=$1; name=$2; extra=$3
tmp=$(mktemp -d)
git archive "$rev" paper_2412_20185_b200/csrc include | tar -x -C "$tmp"
mkdir -p build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -cudart shared $extra \
  -I "$tmp/include" -I "$tmp/paper_2412_20185_b200/csrc" -o "build/libdecdec_$name.so" \
  "$tmp"/paper_2412_20185_b200/csrc/*.cu "$tmp"/paper_2412_20185_b200/csrc/*.cpp
rm -rf "$tmp"
echo "build/libdecdec_$name.so"
