#!/bin/bash
# A/B of variant libraries against the tree: tools/gpu_ab_var.sh "var1 var2" case1 case2 ...
vars=$1; shift
for r in 1 2; do
  echo "tree:"; timeout 120 python tools/prof_block.py "$@" --iters 3 --timed 200 2>&1 | tail -$#
  for v in $vars; do echo "$v:"; WLFUSE_LIB_AB=build/var_$v/libwlfuse.so timeout 120 python tools/prof_block.py "$@" --iters 3 --timed 200 2>&1 | tail -$#; done
done
