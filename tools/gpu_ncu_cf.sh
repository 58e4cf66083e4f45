mkdir -p gpurun_out
for c in cf112 cfs2_112; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"cf" --launch-skip 2 -c 1 \
    -o gpurun_out/ncu_$c -f python tools/prof_block.py $c --iters 3 > gpurun_out/ncu_$c.log 2>&1
done
ls -la gpurun_out/
