mkdir -p gpurun_out
run() { timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 3 -c 1 -o gpurun_out/prof_$1 -f python tools/prof_block.py $3 --iters 3 > /dev/null 2>&1; }
run cf112 cf_fused cf112
run cf56 cf_fused cf56
run mbs2_28 mb_front mbs2_28
run mb14 mb_front mb14
run cfs2 cf2_kernel cfs2_112
timeout 300 python bench.py --skip-cpu > gpurun_out/bench.json 2>/dev/null
