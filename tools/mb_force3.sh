for f in "" "1,2,2,64" "1,1,2,64" "1,2,2,32" "1,2,1,128"; do
  echo "== force '$f'"
  WL_MB_FORCE="$f" python tools/prof_block.py mb7 2>&1 | tail -1
done
