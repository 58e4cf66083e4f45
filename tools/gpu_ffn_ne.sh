#!/bin/bash
# FFN E-ring depth A/B: parity (convnext/ffn), timings NE=2 (variant) vs NE=3 (tree), CTA-0 trace
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_convnext.py tests/test_gpu_parity.py tests/test_big_golden.py -m gpu -x -q -k "convnext or ffn or FFN or cnx" > gpurun_out/pytest_ffn.log 2>&1; echo "rc $?" >> gpurun_out/pytest_ffn.log
tail -3 gpurun_out/pytest_ffn.log
for r in 1 2; do
echo "NE2:"; WLFUSE_LIB_AB=build/var_ne2/libwlfuse.so timeout 120 python tools/prof_block.py cnx96 cnx192 cnx384 cnx768 ffn384 --iters 3 --timed 200 2>&1 | tail -6
echo "NE3:"; timeout 120 python tools/prof_block.py cnx96 cnx192 cnx384 cnx768 ffn384 --iters 3 --timed 200 2>&1 | tail -6
done
timeout 120 python tools/trace_ffn.py 96x56 192x28 2>&1 | tail -40
timeout 300 python tools/bench_convnext.py 128 224 2>&1 | tail -5
