#!/bin/bash
# fresh timing + ncu source-level captures of the stride-1 MBConv blocks
mkdir -p gpurun_out
python tools/prof_block.py mb14 mb7 --iters 1 --timed 200 > gpurun_out/mb_timed.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mb_s1 -s 2 -c 1 -o gpurun_out/ncu_mb7_cur python tools/prof_block.py mb7 --iters 3 --timed 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mb_s1 -s 2 -c 1 -o gpurun_out/ncu_mb14_cur python tools/prof_block.py mb14 --iters 3 --timed 0 > /dev/null 2>&1
cat gpurun_out/mb_timed.txt
