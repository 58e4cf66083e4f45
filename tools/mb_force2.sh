for f in "" "0,2,2,32" "0,1,2,32" "1,2,1,32" "1,1,2,32"; do
  echo "== dxn force '$f'"
  WL_MB_FORCE="$f" python tools/prof_block.py mb14 mb7 2>&1 | tail -2
done
