run() { timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 3 -c 1 -o gpurun_out/prof_$1 -f python tools/prof_block.py $3 --iters 3 > /dev/null 2>&1; }
run cf28 cf_fused cf28
run mb7 mb_front mb7
