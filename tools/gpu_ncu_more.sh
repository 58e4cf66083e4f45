mkdir -p gpurun_out
run() {  # name regex case
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 3 -c 1 -o gpurun_out/prof_$1 -f \
    python tools/prof_block.py $3 --iters 3 > gpurun_out/prof_$1.log 2>&1
}
run cf112 cf_fused cf112
run mb7 mb_front mb7
run mbs2_28 mb_front mbs2_28
run stem stem_kernel stem
run headpool head_pool head
ls gpurun_out/*.ncu-rep
