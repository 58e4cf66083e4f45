#!/bin/bash
# Build build/var_<name>/libwlfuse.so with ONE csrc file taken from a git revision
# (A/B against the working tree): tools/variant_head.sh NAME FILE.cu [REV]
set -e
cd "$(dirname "$0")/.."
name=$1; file=$2; rev=${3:-HEAD}
out=build/var_$name; mkdir -p $out
git show $rev:paper_2404_03617_b200/csrc/$file > paper_2404_03617_b200/csrc/_var_$file
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -Iinclude -Ipaper_2404_03617_b200/csrc -c paper_2404_03617_b200/csrc/_var_$file -o $out/var.o
rm -f paper_2404_03617_b200/csrc/_var_$file
objs=$(ls build/obj/*.o | grep -v "/$(basename $file .cu).o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libwlfuse.so $objs $out/var.o -lcuda
echo built $out/libwlfuse.so
