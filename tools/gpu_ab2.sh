# A/B: build/ab2 (A) vs in-tree (B), alternated
for r in 1 2; do
  echo "A:"; WLFUSE_LIB_AB=build/ab2/libwlfuse.so python tools/prof_block.py "$@" 2>&1 | tail -12
  echo "B:"; python tools/prof_block.py "$@" 2>&1 | tail -12
done
