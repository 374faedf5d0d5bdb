#!/bin/bash
# Builds an A/B variant of libfbgpu.so with extra nvcc defines:
#   tools/build_variant.sh NAME -DFOO=1 ...   ->  build/variants/NAME/libfbgpu.so
# Use with FBGPU_LIB=build/variants/NAME/libfbgpu.so (dev experiments only).
set -e
NAME=$1; shift
HERE=$(cd "$(dirname "$0")/.." && pwd)
SRC=$HERE/paper_2510_14392_b200/csrc
OUT=$HERE/build/variants/$NAME
mkdir -p "$OUT"
FL="-std=c++17 -O3 -lineinfo -fmad=false -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -ffp-contract=off"
nvcc $FL "$@" -c "$SRC/fb_engine.cu" -o "$OUT/fb_engine.o" &
nvcc $FL "$@" -c "$SRC/fb_api.cu" -o "$OUT/fb_api.o" &
nvcc $FL "$@" -c "$SRC/fb_cluster.cu" -o "$OUT/fb_cluster.o" &
g++ -std=c++17 -O2 -fPIC -ffp-contract=off -fno-fast-math -c "$SRC/fb_host.cpp" -o "$OUT/fb_host.o" &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libfbgpu.so" "$OUT/fb_engine.o" "$OUT/fb_cluster.o" "$OUT/fb_api.o" "$OUT/fb_host.o"
echo "$OUT/libfbgpu.so"
