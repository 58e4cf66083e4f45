#!/bin/bash
# Build build/ab/libwlfuse.so from csrc with some files taken from a git
# revision (A/B timing: WLFUSE_LIB_AB=build/ab/libwlfuse.so python tools/prof_block.py ...).
# usage: tools/ab_build.sh REV file.cu [file.cu ...]
set -e
cd "$(dirname "$0")/.."
rev=$1; shift
rm -rf build/ab && mkdir -p build/ab/csrc build/ab/obj
cp paper_2404_03617_b200/csrc/* build/ab/csrc/
mkdir -p build/include && cp include/wlfuse.h build/include/
for f in "$@"; do
  git show "$rev:paper_2404_03617_b200/csrc/$f" > "build/ab/csrc/$f"
  # older revisions predate the stride-1 ConvFirst trace hook
  if [ "$f" = cf_fused.cu ] && ! grep -q cf_set_trace "build/ab/csrc/$f"; then
    echo 'namespace wl { void cf_set_trace(void*) {} }' >> "build/ab/csrc/$f"
  fi
done
for f in build/ab/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
    --expt-relaxed-constexpr -Iinclude -Ipaper_2404_03617_b200/csrc -c "$f" -o "build/ab/obj/$(basename "$f" .cu).o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/libwlfuse.so build/ab/obj/*.o -lcuda
