#!/bin/bash
# new MBConv kernel: parity on the MBConv cases, timeline, then timing new vs legacy
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_big_golden.py -m gpu -x -q -k "mbconv or mb or big" 2>&1 | tail -3
timeout 120 python tools/trace_mb1.py 14 7
timeout 120 python tools/prof_block.py mb14 mb7
WL_MB_LEGACY=1 timeout 120 python tools/prof_block.py mb14 mb7
