# A/B unit times: in-tree library (B) vs build/ab (A), alternated
for r in 1 2; do
  echo "A:"; WLFUSE_LIB_AB=build/ab/libwlfuse.so python tools/prof_block.py "$@" 2>&1 | tail -12
  echo "B:"; python tools/prof_block.py "$@" 2>&1 | tail -12
done
