#!/bin/bash
# Build libhmgpu.so with extra nvcc defines into a separate directory (with a
# copy of libhmbem.so) for A/B timing via HMGPU_LIB_DIR.  Development helper.
# usage: scripts/build_variant.sh <outdir> -DNAME=VALUE ...
set -e
out=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$out"
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
  -Xcompiler -fPIC -Xcompiler -ffp-contract=off -I "$root/include" -shared -cudart static \
  "$@" -o "$out/libhmgpu.so" "$root/paper_2205_04752_b200/csrc/gpu/hmgpu.cu"
cp "$root/paper_2205_04752_b200/lib/libhmbem.so" "$out/"
