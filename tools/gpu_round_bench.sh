#!/bin/bash
# one GPU call: bench (default args), ncu launch list of a short bench, ncu --set full of the top kernels
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --skip-cpu > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cf2_kernel|mb_front|mb_back|cf_fused" -s 4 -c 4 -o gpurun_out/prof_units python tools/prof_block.py cfs2_112 mb14 cf112 --iters 2 > gpurun_out/prof_units.log 2>&1
ls -la gpurun_out
