#!/bin/bash
# Build libtiledqr.so from a source tree into tools/variants/<name>.so (A/B timing aid).
#   tools/build_variant.sh <name> <srcroot> [extra nvcc flags...]
set -e
name=$1; src=$2; shift 2
mkdir -p tools/variants /tmp/vb_$name
for f in trees dag tiledqr; do
  ext=cpp; [ $f = tiledqr ] && ext=cu
  x=""; [ $ext = cpp ] && x="-x c++"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    -I $src/include $x "$@" -c $src/paper_1104_4475_b200/csrc/$f.$ext -o /tmp/vb_$name/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/variants/$name.so /tmp/vb_$name/*.o
echo built tools/variants/$name.so
