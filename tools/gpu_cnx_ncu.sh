#!/bin/bash
# ncu --set full of the ConvNeXt-T hot kernels (one launch each)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_convnext.py -m gpu -x -q > gpurun_out/pytest_cnx.log 2>&1; echo "rc $?" >> gpurun_out/pytest_cnx.log; tail -2 gpurun_out/pytest_cnx.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o gpurun_out/ncu_cnx_stem python tools/prof_block.py cnx_stem --iters 1 --timed 0 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dwln -c 1 -o gpurun_out/ncu_cnx_dwln192 python tools/prof_block.py cnx192 --iters 1 --timed 0 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o gpurun_out/ncu_cnx_exp192 python tools/prof_block.py cnx192 --iters 1 --timed 0 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:cf_fused -c 1 -o gpurun_out/ncu_cnx96 python tools/prof_block.py cnx96 --iters 1 --timed 0 > /dev/null 2>&1
timeout 300 python tools/bench_convnext.py 128 224 > gpurun_out/bench_cnx.txt 2>&1
cat gpurun_out/bench_cnx.txt
ls -la gpurun_out/*.ncu-rep
