mkdir -p gpurun_out
python tools/trace_mb.py mb14 mb7 mbs2 > gpurun_out/trace_mb.txt 2>&1
python tools/prof_block.py mb14 mb7 cf112 cfs2_112 cfs2_56 cf56 cf28 stem head > gpurun_out/unit_times.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mb_front" -s 3 -c 1 -o gpurun_out/prof_mb14 python tools/prof_block.py mb14 --iters 3 > gpurun_out/prof_mb14.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cf2_kernel" -s 3 -c 1 -o gpurun_out/prof_cfs2 python tools/prof_block.py cfs2_112 --iters 3 > gpurun_out/prof_cfs2.log 2>&1
cat gpurun_out/trace_mb.txt gpurun_out/unit_times.txt
