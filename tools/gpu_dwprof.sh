timeout 300 ncu --set full --clock-control none --import-source on -k regex:dwln -s 1 -c 1 -o gpurun_out/ncu_dwln96 python tools/prof_block.py cnx96 --iters 2 --timed 0 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dwln -s 1 -c 1 -o gpurun_out/ncu_dwln384 python tools/prof_block.py cnx384 --iters 2 --timed 0 > /dev/null 2>&1
ls gpurun_out/ncu_dwln*
