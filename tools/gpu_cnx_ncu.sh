#!/bin/bash
# ncu --set full of the ConvNeXt-T hot kernels (one launch each)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_convnext.py tests/test_gpu_parity.py -m gpu -x -q -k "convnext or ffn or golden or gemm" > gpurun_out/pytest_cnx.log 2>&1; echo "rc $?" >> gpurun_out/pytest_cnx.log; tail -2 gpurun_out/pytest_cnx.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cnx_launches.csv python tools/prof_block.py cnx96 --iters 1 --timed 0 > /dev/null 2>&1
grep -E "dwln|ffn_fused" gpurun_out/cnx_launches.csv | awk -F'","' '{print substr($5,1,40), $NF}'
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dwln -c 1 -o gpurun_out/ncu_cnx_dwln192 python tools/prof_block.py cnx192 --iters 1 --timed 0 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ffn_fused -c 1 -o gpurun_out/ncu_cnx_ffn96 python tools/prof_block.py cnx96 --iters 1 --timed 0 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ffn_fused -c 1 -o gpurun_out/ncu_cnx_ffn192 python tools/prof_block.py cnx192 --iters 1 --timed 0 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
