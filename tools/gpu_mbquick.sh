#!/bin/bash
# MBConv kernel iteration: parity subset, block timings, CTA-0 trace
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_big_golden.py tests/test_gpu_layerwise.py -q -x -k "mb or MBConv or mbconv or stage or network or golden" > gpurun_out/pytest_mbq.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_mbq.log
timeout 120 python tools/prof_block.py mb14 mb7 --iters 3 --timed 200 > gpurun_out/mb_timed.txt 2>&1
timeout 120 python tools/trace_mb1.py 14 7 > gpurun_out/trace_mb1.txt 2>&1
tail -4 gpurun_out/pytest_mbq.log; cat gpurun_out/mb_timed.txt gpurun_out/trace_mb1.txt
